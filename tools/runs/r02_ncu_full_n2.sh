#!/bin/bash
# ncu --set full of one copy_tiles launch (256-bit peer stores) in the N=2 balanced
# placement, one process driving 2 GPUs (gpurun --gpus 2): gpurun_out/r02nf/.
O=gpurun_out/r02nf; mkdir -p $O
CUDA_VISIBLE_DEVICES=0,1 timeout 300 python tools/p2p_profile.py --layers 8 --reps 2 --gpus 2 --placement balanced > $O/live.json 2> $O/live.err && \
CUDA_VISIBLE_DEVICES=0,1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:copy_tiles -c 1 \
    -o $O/copy_tiles_n2_balanced python tools/p2p_profile.py --layers 8 --reps 1 --gpus 2 --placement balanced > $O/ncu.out 2>&1
ncu -i $O/copy_tiles_n2_balanced.ncu-rep --page raw --csv > $O/raw.csv 2> $O/raw.err
