# one GPU session: smoke, parity tests, bench (C2), launch list, ncu captures of the fast, dense and Selector kernels
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -3 gpurun_out/bench_c2.err; cat gpurun_out/bench_c2.json
timeout 600 python bench.py --impl reference --steps 8 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
# launch list of 2 timed steps (one fast graph + kernels of a slow one): skip the setup kernels
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 6 --warmup 3 --no-cpu --no-e2e --no-graph > /dev/null 2>&1; echo ncu1 $?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fast_decode -s 40 -c 1 -o gpurun_out/prof_fast python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-graph > gpurun_out/ncu2.log 2>&1; echo ncu2 $?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 2 -c 1 -o gpurun_out/prof_dense python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-graph > gpurun_out/ncu3.log 2>&1; echo ncu3 $?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sel_ -s 0 -c 4 -o gpurun_out/prof_selector python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-graph > gpurun_out/ncu4.log 2>&1; echo ncu4 $?
