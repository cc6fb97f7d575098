# one GPU session: parity tests, bench, launch list, ncu captures of the decode + selector kernels
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -3 gpurun_out/bench_c2.err; cat gpurun_out/bench_c2.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo ncu1 $?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 36 -c 1 -o gpurun_out/prof_sparse python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-graph > gpurun_out/ncu2.log 2>&1; echo ncu2 $?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 0 -c 1 -o gpurun_out/prof_dense python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-graph > gpurun_out/ncu3.log 2>&1; echo ncu3 $?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sel_ -s 0 -c 3 -o gpurun_out/prof_selector python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-graph > gpurun_out/ncu4.log 2>&1; echo ncu4 $?
