# round-2 evidence in one GPU session: launch lists (C2, C4), ncu --set full of the tcgen05 dense decode and the
# long-row top-k, compute-sanitizer over the round-2 kernels (K1-TC, the long-row top-k, the Selector stages,
# the C++ executor)
export PYTHONPATH=$GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02
O=gpurun_out/r02
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
# launch lists: 6 timed steps (eager, so each kernel is a separate launch), setup kernels included
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv \
  python bench.py --steps 6 --warmup 3 --no-cpu --no-e2e --no-graph > /dev/null 2>&1; echo ncu-c2 $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv \
  python bench.py --config c4 --steps 4 --warmup 3 --no-cpu --no-e2e --no-graph > /dev/null 2>&1; echo ncu-c4 $?
timeout 400 ncu --set full --clock-control none --import-source on -k regex:decode_tc -s 2 -c 1 -o $O/prof_dense_tc_c4 \
  python bench.py --config c4 --steps 2 --warmup 3 --no-cpu --no-e2e --no-graph > $O/ncu_tc.log 2>&1; echo ncu-tc $?
timeout 400 ncu --set full --clock-control none --import-source on -k regex:sel_bt -s 0 -c 4 -o $O/prof_bt_c4 \
  python bench.py --config c4 --steps 2 --warmup 3 --no-cpu --no-e2e --no-graph > $O/ncu_bt.log 2>&1; echo ncu-bt $?
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 1200 compute-sanitizer --tool $tool --print-limit 6 python -m pytest tests/test_decode_tc.py \
    tests/test_selector_stages.py tests/test_executor.py -m gpu -q -p no:cacheprovider 2>&1 \
    | grep -vE "Host Frame|^=========\s*$" | tail -5
  timeout 900 compute-sanitizer --tool $tool --print-limit 6 python -m pytest tests/test_baseline_parity.py -m gpu -q \
    -p no:cacheprovider -k "long_row and False" 2>&1 | grep -vE "Host Frame|^=========\s*$" | tail -5
done 2>&1 | tee $O/sanitizer.txt
