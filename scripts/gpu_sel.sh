for c in 2 4 8; do echo "C=$c"; SFI_FAST_CLUSTER=$c timeout 300 python scripts/microbench_decode.py --layers 36 --iters 40 2>&1 | tail -1; done
