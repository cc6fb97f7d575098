timeout 300 python scripts/microbench_decode.py --layers 36 --iters 40 2>&1 | tail -1
