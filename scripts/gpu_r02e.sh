export PYTHONPATH=$GRAFT_REPO_ROOT
O=gpurun_out/r02
mkdir -p $O
timeout 900 python -m pytest tests/test_baseline_parity.py -m gpu -x -q 2>&1 | tail -3
SFI_TOPK_BT=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_selector_stages.py -m gpu -x -q -k "selector or ties or stage" 2>&1 | tail -3
SFI_TOPK_BT=1 timeout 300 python scripts/probe_topk.py c3 c4 2>&1 | tail -2
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --config c3 --also c4 > $O/bench_bt_e.json 2> $O/bench_bt_e.err; echo bench $?
