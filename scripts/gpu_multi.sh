# 2 ranks on one GPU over gloo (functional check of the N>1 bench paths; not a measurement)
for cfg in c2 c3; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 4 --warmup 3 --config $cfg --layers 2 --no-graph --backend gloo --no-cpu 2>&1 | tail -3
done
