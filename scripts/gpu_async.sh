timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
SFI_TOPK_P16=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "selector or async or prefill" 2>&1 | tail -2
for k in 1 0; do SFI_TOPK_P16=$k timeout 300 python scripts/microbench_decode.py --layers 4 --iters 12 2>&1 | tail -2 | head -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('p16=$k', 'selector', d['selector_us'])"; done
for k in 1 0; do SFI_TOPK_P16=$k timeout 600 python bench.py --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('p16=$k', d['value'], d['ms_per_step'])"; done
