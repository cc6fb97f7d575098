timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('async', d['value'], d['ms_per_step'], d['e2e']['value'], d['kernels']['dense_decode'])"
timeout 600 python bench.py --no-cpu --no-e2e --sync-slow 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sync', d['value'], d['ms_per_step'])"
