export PYTHONPATH=$GRAFT_REPO_ROOT
O=gpurun_out/r02/share
mkdir -p $O
run() {  # name, config, env...
  n=$1; cfg=$2; shift 2
  env "$@" timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu --no-e2e --also none > $O/$n.json 2> $O/$n.err
  python -c "import json,sys; d=json.loads(open('$O/$n.json').read().strip().splitlines()[-1]); print('$n', round(d['value'],1), round(d['slow_step_us_graph']), round(d['fast_step_us_graph']))" 2>/dev/null || tail -2 $O/$n.err
}
for c in c2 c3 c4; do for sl in 1 2 3 4; do run ${c}_slots$sl $c SFI_EXEC_SLOTS=$sl; done; done
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02/bench_default_j.json 2> gpurun_out/r02/bench_default_j.err; echo bench $?
