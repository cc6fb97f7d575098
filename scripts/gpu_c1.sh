SFI_DECODE_TRACE=1 timeout 300 python scripts/microbench_decode.py --layers 4 --batch 1 --ctx 8192 --hq 16 2>&1 | grep -A3 "^\[dense\]" | head -3
timeout 300 python scripts/microbench_decode.py --layers 28 --batch 1 --ctx 8192 --hq 16 --iters 40 2>&1 | tail -1 | cut -c1-300
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "dense" 2>&1 | tail -1
timeout 600 python bench.py --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['value'], d['kernels']['dense_decode']['ms'])"
timeout 600 python bench.py --config c1 --steps 64 --warmup 4 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1', d['value'], d['kernels']['dense_decode']['ms'])"
