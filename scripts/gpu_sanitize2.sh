export PYTHONPATH=$GRAFT_REPO_ROOT
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 1500 compute-sanitizer --tool $tool --print-limit 6 python -m pytest tests/test_seq_sharded.py tests/test_sharded.py -m gpu -q -p no:cacheprovider -k "lockstep or one_gpu or simulated" --deselect "tests/test_seq_sharded.py::test_sequence_sharded_two_processes_one_gpu" --deselect "tests/test_sharded.py::test_head_sharded_two_processes_one_gpu" 2>&1 | grep -vE "Host Frame|^=========\s*$" | tail -5
done
