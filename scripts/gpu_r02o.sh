export PYTHONPATH=$GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02
run() { n=$1; c=$2; shift 2; env "$@" timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e --also none > gpurun_out/r02/b.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r02/b.json').read().strip().splitlines()[-1]); print('$n', round(d['value'],1), round(d['slow_step_us_graph']))"; }
for pm in 500 650 675 750 875 1000; do run c1_$pm c1 SFI_DENSE_SHARE_PERMILLE=$pm; done
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02/bench_o.json 2> gpurun_out/r02/bench_o.err; echo bench $?
