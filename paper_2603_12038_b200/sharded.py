"""Multi-GPU SFI decode: one process per GPU, torch.distributed for
the plumbing (NCCL over NVLink on B200 boxes; gloo for CPU-side tests).

KV-head sharding (config C3): rank r of P holds KV heads [r*H/P, (r+1)*H/P) of
every layer and request (and their G query heads each). Attention, key norms,
the ring, the compact builder and every Selector stage except cross-head
exclusivity are per head, so fast steps exchange nothing. Cross-head
exclusivity (selector.cpp:204-230) is a softmax over all KV heads of a request
at each position: per layer and slow step the ranks all-gather the Selector's
z_base blocks (fp64 [B][H/P][max_positions]) and each finishes soft-NMS +
cross-head in global head order and the top-k of its own heads — indices
bit-identical to the 1-GPU Selector.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .device import SfiCache


def head_range(n_kv_heads: int, world: int, rank: int) -> tuple[int, int]:
    """KV heads owned by `rank` (contiguous, equal blocks)."""
    if n_kv_heads % world != 0:
        raise ValueError(f"{n_kv_heads} KV heads do not split over {world} ranks")
    per = n_kv_heads // world
    return rank * per, (rank + 1) * per


def all_gather_blocks(local: torch.Tensor, out: torch.Tensor, group=None) -> torch.Tensor:
    """out[r] = local of rank r (rank order). NCCL gathers in place on the current
    stream; gloo (CPU tests) stages CUDA tensors through host memory."""
    backend = dist.get_backend(group)
    if backend == "nccl" or not local.is_cuda:
        dist.all_gather_into_tensor(out.view(-1), local.contiguous().view(-1), group=group)
        return out
    host = torch.empty_like(out, device="cpu")
    dist.all_gather_into_tensor(host.view(-1), local.detach().cpu().contiguous().view(-1), group=group)
    out.copy_(host)
    return out


class HeadShardedSfi:
    """This rank's shard of a KV-head-sharded SFI cache (n_layers x batch x
    n_kv_heads/P heads). Same step API as SfiCache; only the Selector talks to
    the other ranks."""

    def __init__(self, n_layers: int, batch: int, n_kv_heads: int, n_q_heads: int, head_dim: int,
                 max_positions: int, n_sink: int = 4, k_budget: int = 2048, n_recent: int = 256,
                 group=None, device=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.h0, self.h1 = head_range(n_kv_heads, self.world, self.rank)
        G = n_q_heads // n_kv_heads
        self.n_kv_heads, self.n_q_heads, self.G = n_kv_heads, n_q_heads, G
        self.local_heads = self.h1 - self.h0
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.cache = SfiCache(n_layers, batch, self.local_heads, self.local_heads * G, head_dim,
                              max_positions, n_sink, k_budget, n_recent, device=device)
        dev = self.cache.k_cache.device
        self.z_all = torch.empty((self.world, batch, self.local_heads, max_positions), dtype=torch.float64,
                                 device=dev)

    # q heads of this shard: [h0*G, h1*G) of the model's q heads
    def q_slice(self) -> slice:
        return slice(self.h0 * self.G, self.h1 * self.G)

    def selector(self, layer: int, logits: torch.Tensor, params=None):
        z = self.cache.selector_fuse(layer, logits, params)
        if self.world > 1:
            all_gather_blocks(z, self.z_all, self.group)
            self.cache.selector_finish(layer, self.z_all, self.world, self.rank, params)
        else:
            self.cache.selector_finish(layer, z.unsqueeze(0), 1, 0, params)

    def __getattr__(self, name):  # everything else is per head: the local cache
        return getattr(self.cache, name)
