# aux (Selector) stream at high priority, dense over-decomposed so freed slots go to the Selector first
export PYTHONPATH=$GRAFT_REPO_ROOT
O=gpurun_out/r02/prio; mkdir -p $O
run() {  # name, config, env...
  n=$1; cfg=$2; shift 2
  env "$@" timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu --no-e2e --also none > $O/$n.json 2> $O/$n.err
  python -c "import json,sys; d=json.loads(open('$O/$n.json').read().strip().splitlines()[-1]); print('$n', round(d['value'],1), round(d['slow_step_us_graph']), round(d['fast_step_us_graph']))" 2>/dev/null || tail -2 $O/$n.err
}
for c in c2 c3; do
run ${c}_default $c
run ${c}_prio2 $c SFI_EXEC_PRIO=2
run ${c}_prio2_full $c SFI_EXEC_PRIO=2 SFI_DENSE_SHARE_PERMILLE=1000
run ${c}_prio2_592 $c SFI_EXEC_PRIO=2 SFI_DECODE_CTAS=592
run ${c}_prio2_1024 $c SFI_EXEC_PRIO=2 SFI_DECODE_CTAS=1024
run ${c}_prio0_592 $c SFI_DECODE_CTAS=592
done
