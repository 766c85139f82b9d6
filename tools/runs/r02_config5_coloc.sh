#!/bin/bash
# Config 5 (Llama-3-70B TP4xPP2 -> TP8) at the full model's per-GPU state (N=4, L=40) under
# 180 GB per GPU with the balanced co-location (gpurun --gpus 4): gpurun_out/r02c5/.
O=gpurun_out/r02c5; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 1500 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4 --master-port 29995 \
    tools/configs_bench.py --config 5 --layers 40 --arena-cap 180 --placement balanced --reps 3 > $O/config5_balanced.jsonl 2> $O/config5_balanced.err
