# fast-step cluster size at the small-slice configs (C1: 8 slices, C4: 4 slices)
export PYTHONPATH=$GRAFT_REPO_ROOT; mkdir -p gpurun_out/r02
run() { n=$1; c=$2; shift 2; env "$@" timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e --also none > gpurun_out/r02/b.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r02/b.json').read().strip().splitlines()[-1]); print('$n', round(d['value'],1), round(d['fast_step_us_graph'],1))"; }
for C in 0 4 6 8 12; do run c4_C$C c4 SFI_FAST_CLUSTER=$C; done
for C in 0 4 8 12; do run c1_C$C c1 SFI_FAST_CLUSTER=$C; done
