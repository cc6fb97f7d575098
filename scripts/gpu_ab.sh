# A/B: parity tests, then bench with PDL on and off (no CPU leg)
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for pdl in 1 0; do SFI_PDL=$pdl timeout 600 python bench.py --no-cpu > gpurun_out/bench_pdl$pdl.json 2>gpurun_out/bench_pdl$pdl.err; tail -2 gpurun_out/bench_pdl$pdl.err; done
