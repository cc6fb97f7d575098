timeout 600 python scripts/microbench_decode.py --layers 1 --batch 288 --ctx 32768 --iters 8 2>&1 | tail -2 | cut -c1-400
