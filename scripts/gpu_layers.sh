SFI_LAYER_TRACE=1 timeout 300 python scripts/probe_layers.py 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fast or sparse" 2>&1 | tail -2
timeout 600 python bench.py --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['kernels']['fast_decode']['ms'], d['kernels']['fast_decode']['frac'])"
