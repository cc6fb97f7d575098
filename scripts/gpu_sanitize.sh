export PYTHONPATH=$GRAFT_REPO_ROOT
for k in "fast_decode_fused" "group16" "sparse_decode_vs"; do
  echo "== $k"
  timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 4 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "$k" -p no:cacheprovider 2>&1 | grep -vE "Host Frame|^=========\s*$" | grep -E "hazard|Write|Read|at |RACECHECK|kernel|passed|failed" | head -24
done
