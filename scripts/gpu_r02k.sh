export PYTHONPATH=$GRAFT_REPO_ROOT
O=gpurun_out/r02/share; mkdir -p $O
run() {  # name, config, env...
  n=$1; cfg=$2; shift 2
  env "$@" timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu --no-e2e --also none > $O/$n.json 2> $O/$n.err
  python -c "import json,sys; d=json.loads(open('$O/$n.json').read().strip().splitlines()[-1]); print('$n', round(d['value'],1), round(d['slow_step_us_graph']), round(d['fast_step_us_graph']), d['roofline'].get('grid'))" 2>/dev/null || tail -2 $O/$n.err
}
for rep in 1 2; do
run c3_default_$rep c3
run c3_env750_$rep c3 SFI_DENSE_SHARE_PERMILLE=750
run c3_env750_tc0_$rep c3 SFI_DENSE_SHARE_PERMILLE=750 SFI_DENSE_TC=1
done
