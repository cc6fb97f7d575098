# ncu --set full of C1's in-step dense decode (mma.sync share grid) for bench.py's roofline.traffic
export PYTHONPATH=$GRAFT_REPO_ROOT
O=gpurun_out/r02f; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:decode_kernel" -s 6 -c 1 -o $O/prof_dense_c1 \
  python bench.py --config c1 --steps 2 --warmup 3 --no-cpu --no-e2e --no-graph --also none > $O/ncu_c1.log 2>&1; echo p-c1 $?
