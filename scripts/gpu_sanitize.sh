# compute-sanitizer memcheck + racecheck + synccheck over the GPU parity suite (small shapes)
export PYTHONPATH=$GRAFT_REPO_ROOT
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 1500 compute-sanitizer --tool $tool --print-limit 10 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "not C2 and not 32768" 2>&1 | grep -vE "Host Frame|^=========\s*$" | tail -6
done
