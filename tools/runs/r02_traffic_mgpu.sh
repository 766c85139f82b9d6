#!/bin/bash
# DRAM traffic of the N>1 forward launch with the round-2 kernel (256-bit peer stores), one
# process driving 2 / 4 GPUs (gpurun --gpus 4): outputs under gpurun_out/r02tm/.
O=gpurun_out/r02tm; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 600 python tools/p2p_profile.py --layers 32 --reps 3 --gpus 2 > $O/live_n2.json 2> $O/live_n2.err
timeout 600 python tools/p2p_profile.py --layers 32 --reps 3 --gpus 4 > $O/live_n4.json 2> $O/live_n4.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
CUDA_VISIBLE_DEVICES=0,1 timeout 1200 ncu --replay-mode application --metrics $M --clock-control none -k regex:copy_tiles -c 2 --csv \
    --log-file $O/ncu_n2.csv python tools/p2p_profile.py --layers 32 --reps 1 --gpus 2 > $O/ncu_n2.out 2>&1
timeout 1200 ncu --replay-mode application --metrics $M --clock-control none -k regex:copy_tiles -c 4 --csv \
    --log-file $O/ncu_n4.csv python tools/p2p_profile.py --layers 32 --reps 1 --gpus 4 > $O/ncu_n4.out 2>&1
