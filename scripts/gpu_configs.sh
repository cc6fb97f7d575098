timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_seq_sharded.py -m gpu -x -q 2>&1 | tail -2
for cfg in c1 c3 c4; do
  timeout 1200 python bench.py --config $cfg --steps 64 --warmup 4 --no-cpu > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err; echo "$cfg rc=$?"; tail -2 gpurun_out/bench_$cfg.err
done
