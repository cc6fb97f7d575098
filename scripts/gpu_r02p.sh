export PYTHONPATH=$GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02
run() { n=$1; c=$2; shift 2; env "$@" timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e --also none > gpurun_out/r02/b.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r02/b.json').read().strip().splitlines()[-1]); print('$n', round(d['value'],1), round(d['slow_step_us_graph']))"; }
run c2_mma675 c2
for pm in 550 600 650 700 725; do run c2_tc3_$pm c2 SFI_DENSE_TC_SHARE_G=4 SFI_DENSE_TC_SHARE_PERMILLE=$pm; done
run c3_mma750 c3
for pm in 650 700 725; do run c3_tc3_$pm c3 SFI_DENSE_TC_SHARE_G=8 SFI_DENSE_TC_SHARE_PERMILLE=$pm; done
