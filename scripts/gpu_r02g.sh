# C3 / C2 async slow step: mma.sync share grid vs tcgen05 beside the Selector (grid share, stages)
export PYTHONPATH=$GRAFT_REPO_ROOT
O=gpurun_out/r02/share
mkdir -p $O
run() {  # name, config, env...
  n=$1; cfg=$2; shift 2
  env "$@" timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu --no-e2e --also none > $O/$n.json 2> $O/$n.err
  python -c "import json,sys; d=json.loads(open('$O/$n.json').read().strip().splitlines()[-1]); print('$n', round(d['value'],1), round(d['slow_step_us_graph']), round(d['roofline']['ms'] if 'ms' in d['roofline'] else 0,3))" 2>/dev/null || tail -2 $O/$n.err
}
run c3_mma c3
run c3_tc1000_2 c3 SFI_DENSE_TC_SHARE_G=8
run c3_tc1000_3 c3 SFI_DENSE_TC_SHARE_G=8 SFI_DENSE_TC_SHARE_STAGES=3
run c3_tc750_3 c3 SFI_DENSE_TC_SHARE_G=8 SFI_DENSE_TC_SHARE_STAGES=3 SFI_DENSE_TC_SHARE_PERMILLE=750
run c3_tc850_3 c3 SFI_DENSE_TC_SHARE_G=8 SFI_DENSE_TC_SHARE_STAGES=3 SFI_DENSE_TC_SHARE_PERMILLE=850
run c3_mma800 c3 SFI_DENSE_SHARE_PERMILLE=800
run c3_mma500 c3 SFI_DENSE_SHARE_PERMILLE=500
run c2_mma c2
run c2_tc1000_3 c2 SFI_DENSE_TC_SHARE_G=4 SFI_DENSE_TC_SHARE_STAGES=3
run c2_tc850_3 c2 SFI_DENSE_TC_SHARE_G=4 SFI_DENSE_TC_SHARE_STAGES=3 SFI_DENSE_TC_SHARE_PERMILLE=850
