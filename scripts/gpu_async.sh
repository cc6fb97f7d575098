timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for k in 1 0; do SFI_FAST_PUSH=$k timeout 300 python scripts/microbench_decode.py --layers 36 --iters 40 2>&1 | tail -1 | cut -c1-120; done
for k in 1 0; do SFI_FAST_PUSH=$k timeout 600 python bench.py --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('push=$k', d['value'], d['ms_per_step'], d['e2e']['value'], d['kernels']['fast_decode']['ms'], d['kernels']['fast_decode']['frac'])"; done
