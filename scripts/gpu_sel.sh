timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
SFI_SELECTOR_3K=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k selector 2>&1 | tail -2
for k in 0 1; do SFI_SELECTOR_3K=$k timeout 300 python scripts/microbench_decode.py --layers 4 --iters 12 2>&1 | tail -2 | head -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('legacy' if $k else 'new', 'selector', d['selector_us'])"; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sel_ -s 0 -c 3 -o gpurun_out/prof_selector2 python scripts/microbench_decode.py --layers 1 --iters 4 > /dev/null 2>&1; echo ncu $?
