# round-2 follow-up: new GPU tests, launch lists of the headline step alone, ncu of the C2 Selector chain,
# the C5 line
export PYTHONPATH=$GRAFT_REPO_ROOT
O=gpurun_out/r02
mkdir -p $O
timeout 900 python -m pytest tests/test_generation.py tests/test_gpu_parity.py -m gpu -x -q -k "generation or overflow" 2>&1 | tail -15
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2_only.csv \
  python bench.py --steps 6 --warmup 3 --no-cpu --no-e2e --no-graph --also none > /dev/null 2>&1; echo ncu-c2 $?
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4_only.csv \
  python bench.py --config c4 --steps 4 --warmup 3 --no-cpu --no-e2e --no-graph --also none > /dev/null 2>&1; echo ncu-c4 $?
timeout 400 ncu --set full --clock-control none --import-source on -k "regex:sel_|compact" -s 8 -c 5 -o $O/prof_sel_c2 \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-graph --also none > $O/ncu_sel.log 2>&1; echo ncu-sel $?
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --also c5 > $O/bench_c5.json 2> $O/bench_c5.err; echo c5 $?; tail -3 $O/bench_c5.err
