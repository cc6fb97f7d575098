"""Summaries of ncu captures for profiles/: per-kernel key metrics from `ncu -i X.ncu-rep
--page raw --csv`, and per-kernel launch statistics from a `--metrics gpu__time_duration.sum`
launch list.

    python scripts/ncu_summary.py raw  OUT.json  A.raw.csv [B.raw.csv ...]
    python scripts/ncu_summary.py launches OUT.json LAUNCHES.csv
"""
from __future__ import annotations

import collections
import csv
import io
import json
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio"]


def raw(out, files):
    res = []
    for f in files:
        rows = list(csv.reader(open(f)))
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            d = {"kernel": r[hdr.index("Kernel Name")], "capture": f}
            for k in KEYS:
                if k in hdr:
                    v = r[hdr.index(k)].replace(",", "")
                    try:
                        d[k] = float(v)
                    except ValueError:
                        d[k] = v
                    d[k + ".unit"] = units[hdr.index(k)]
            res.append(d)
    json.dump(res, open(out, "w"), indent=1)
    for d in res:
        print(f"{d.get('gpu__time_duration.sum', 0):10.2f} {d.get('gpu__time_duration.sum.unit', '')}  "
              f"dram {d.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 0):5.1f}%  "
              f"issue {d.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):5.1f}%  {d['kernel'][:80]}")


def launches(out, f):
    txt = open(f).read()
    lines = [ln for ln in txt.splitlines() if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
    agg = collections.OrderedDict()
    for r in rows:
        a = agg.setdefault(r["Kernel Name"], [0, 0.0, []])
        a[0] += 1
        v = float(r["Metric Value"])
        a[1] += v
        a[2].append(v)
    unit = rows[0]["Metric Unit"] if rows else ""
    tot = sum(a[1] for a in agg.values())
    res = {"source": f, "unit": unit, "launches": len(rows), "kernels": [
        {"kernel": k, "count": c, "avg": t / c, "min": min(v), "max": max(v), "share": t / tot}
        for k, (c, t, v) in sorted(agg.items(), key=lambda x: -x[1][1])]}
    json.dump(res, open(out, "w"), indent=1)
    for k in res["kernels"][:20]:
        print(f"{k['count']:6d} {k['avg'] / 1e3:10.2f} us {k['share']:6.3f}  {k['kernel'][:90]}")


if __name__ == "__main__":
    mode, out, *files = sys.argv[1:]
    raw(out, files) if mode == "raw" else launches(out, files[0])
