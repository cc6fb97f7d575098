# compute-sanitizer over the round-2 kernels on the final code: tcgen05 dense decode, Selector stages, the
# executor (graph-replayed steps), a generation, the long-row top-k (forced at short rows too)
export PYTHONPATH=$GRAFT_REPO_ROOT
O=gpurun_out/r02f; mkdir -p $O
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 1500 compute-sanitizer --tool $tool --print-limit 6 python -m pytest tests/test_decode_tc.py \
    tests/test_selector_stages.py tests/test_executor.py tests/test_generation.py -m gpu -q -p no:cacheprovider 2>&1 \
    | grep -vE "Host Frame|^=========\s*$" | tail -4
  SFI_TOPK_BT=1 timeout 900 compute-sanitizer --tool $tool --print-limit 6 python -m pytest tests/test_gpu_parity.py \
    -m gpu -q -p no:cacheprovider -k "selector_indices" 2>&1 | grep -vE "Host Frame|^=========\s*$" | tail -4
done 2>&1 | tee $O/sanitizer.txt
