#!/bin/bash
# N=2 (balanced co-location): one mixed launch vs peer-bound and local tiles as two
# concurrent launches (RS_SPLIT_REMOTE). gpurun --gpus 2; outputs under gpurun_out/r02sp/.
O=gpurun_out/r02sp; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 $TR --nproc-per-node 2 --master-port 29981 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > $O/A.json 2> $O/A.err
RS_SPLIT_REMOTE=1 timeout 300 $TR --nproc-per-node 2 --master-port 29982 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > $O/B.json 2> $O/B.err
RS_SPLIT_REMOTE=1 RS_REMOTE_CTAS_PER_SM=1 timeout 300 $TR --nproc-per-node 2 --master-port 29983 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > $O/C.json 2> $O/C.err
