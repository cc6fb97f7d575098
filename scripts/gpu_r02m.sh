export PYTHONPATH=$GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests/test_baseline_parity.py -m gpu -x -q 2>&1 | tail -2
SFI_TOPK_BT=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_selector_stages.py tests/test_generation.py -m gpu -x -q -k "selector or ties or stage or generation" 2>&1 | tail -2
SFI_TOPK_BT=1 timeout 300 python scripts/probe_topk.py c2 c3 c4 2>&1 | tail -3
for c in c3 c4; do timeout 300 python scripts/probe_pipeline.py $c 2>&1 | head -1; done
for c in c3 c4; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e --also none > gpurun_out/r02/b.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r02/b.json').read().strip().splitlines()[-1]); print('$c', round(d['value'],1), round(d['slow_step_us_graph']))"; done
