timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
timeout 300 python scripts/microbench_decode.py --layers 36 --iters 40 2>&1 | tail -2 | head -1
