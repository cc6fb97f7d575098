export PYTHONPATH=$GRAFT_REPO_ROOT
timeout 1500 compute-sanitizer --tool synccheck --print-limit 4 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "not C2 and not 32768" 2>&1 | grep -vE "Host Frame|^=========\s*$" | grep -E "Error|error|at |passed|failed|SUMMARY" | head -12
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['kernels']['fast_decode']['ms'], d['kernels']['dense_decode']['ms'])"
