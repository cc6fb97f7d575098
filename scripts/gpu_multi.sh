# 2 ranks on one GPU over gloo (functional check of the N>1 bench paths; not a measurement)
for cfg in c3 c4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 4 --warmup 3 --config $cfg --layers 2 --no-graph --backend gloo --no-cpu 2>&1 | tail -2 | cut -c1-600
done
# 1 GPU, full C4 (Qwen3-235B shapes, 94 layers, 256K)
timeout 900 python bench.py --config c4 --steps 64 --warmup 4 --no-cpu 2>&1 | tail -2
