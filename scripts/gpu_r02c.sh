# long-row top-k rework: parity (ties, full-layer C3 / C4, forced at C2 sizes) and timing with / without
export PYTHONPATH=$GRAFT_REPO_ROOT
O=gpurun_out/r02
mkdir -p $O
timeout 900 python -m pytest tests/test_baseline_parity.py -m gpu -x -q 2>&1 | tail -4
SFI_TOPK_BT=1 timeout 900 python -m pytest tests/test_baseline_parity.py tests/test_gpu_parity.py -m gpu -x -q -k "selector or ties or c2" 2>&1 | tail -4
SFI_TOPK_BT=0 timeout 300 python scripts/probe_topk.py c2 c3 c4 2>&1 | tail -3
SFI_TOPK_BT=1 timeout 300 python scripts/probe_topk.py c2 c3 c4 2>&1 | tail -3
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --also c3,c4,c5 > $O/bench_bt0.json 2> $O/bench_bt0.err; echo bench $?
SFI_TOPK_BT=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --also none > $O/bench_bt1.json 2> $O/bench_bt1.err; echo bench-bt1 $?
