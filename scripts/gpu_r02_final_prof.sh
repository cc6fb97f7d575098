# final round-2 evidence: launch lists of the headline step (C2) and C4, ncu --set full of the in-step dense
# decode (the mma.sync share grid) and of the C4 tcgen05 dense decode
export PYTHONPATH=$GRAFT_REPO_ROOT
O=gpurun_out/r02f; mkdir -p $O
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv \
  python bench.py --steps 6 --warmup 3 --no-cpu --no-e2e --no-graph --also none > /dev/null 2>&1; echo l-c2 $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv \
  python bench.py --config c4 --steps 4 --warmup 3 --no-cpu --no-e2e --no-graph --also none > /dev/null 2>&1; echo l-c4 $?
timeout 400 ncu --set full --clock-control none --import-source on -k "regex:decode_kernel" -s 6 -c 1 -o $O/prof_dense_c2 \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-graph --also none > $O/ncu_dense.log 2>&1; echo p-c2 $?
timeout 400 ncu --set full --clock-control none --import-source on -k "regex:decode_tc_kernel" -s 6 -c 1 -o $O/prof_dense_tc_c4 \
  python bench.py --config c4 --steps 2 --warmup 3 --no-cpu --no-e2e --no-graph --also none > $O/ncu_tc.log 2>&1; echo p-c4 $?
