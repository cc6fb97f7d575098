# tuning session: parity tests + per-kernel microbench with CTA timelines + selector ncu
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
SFI_DECODE_TRACE=1 timeout 300 python scripts/microbench_decode.py 2>&1 | grep -v "slow cta"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sel_ -s 0 -c 3 -o gpurun_out/prof_selector python scripts/microbench_decode.py --layers 1 --iters 4 > /dev/null 2>&1; echo ncu $?
