export PYTHONPATH=$GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02
run() { n=$1; c=$2; shift 2; env "$@" timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e --also none > gpurun_out/r02/b.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r02/b.json').read().strip().splitlines()[-1]); print('$n', round(d['value'],1), round(d['slow_step_us_graph']))"; }
for rep in 1 2; do
for pm in 1000 925 850 775 700; do run c4_tc3_$pm c4 SFI_DENSE_TC_SHARE_PERMILLE=$pm; done
run c4_mma_650 c4 SFI_DENSE_TC_SHARE_G=32 SFI_DENSE_SHARE_PERMILLE=650
run c4_mma_1000 c4 SFI_DENSE_TC_SHARE_G=32 SFI_DENSE_SHARE_PERMILLE=1000
done
