# decode timeline study: per-CTA traces at several grid sizes
for n in 296 148 592; do echo "== ctas $n"; SFI_DECODE_CTAS=$n SFI_DECODE_TRACE=1 timeout 300 python scripts/microbench_decode.py --layers 4 2>&1 | grep -v "slow cta"; done
echo "== no trace"; timeout 300 python scripts/microbench_decode.py --layers 4
echo "== batch 32 (4x the bytes)"; timeout 300 python scripts/microbench_decode.py --layers 2 --batch 32 --ctx 8192
