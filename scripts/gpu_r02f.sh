export PYTHONPATH=$GRAFT_REPO_ROOT
O=gpurun_out/r02
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_baseline_parity.py -m gpu -x -q -k "selector or ties or top_k or c2" 2>&1 | tail -3
timeout 300 python scripts/probe_topk.py c2 c1 2>&1 | tail -2
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --also none > $O/bench_f.json 2> $O/bench_f.err; echo bench $?
