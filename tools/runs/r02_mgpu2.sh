#!/bin/bash
# Round-2 multi-GPU batch 2 (gpurun --gpus 4): outputs under gpurun_out/r02m2/.
O=gpurun_out/r02m2; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
CUDA_VISIBLE_DEVICES=0 RS_TIMING=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_n1.json 2> $O/bench_n1.err
timeout 600 $TR --nproc-per-node 4 --master-port 29701 bench.py --gpus 4 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_n4.json 2> $O/bench_n4.err
timeout 900 $TR --nproc-per-node 4 --master-port 29702 tools/configs_bench.py --config 5 --layers 40 --arena-cap 180 --reps 2 > $O/config5_n4_L40_cap180.json 2> $O/config5.err
timeout 600 $TR --nproc-per-node 4 --master-port 29703 bench.py --gpus 4 --steps 5 --warmup 3 --no-cpu-baseline --arena-multi --hbm-cap 45000000000 > $O/bench_n4_arena45.json 2> $O/bench_n4_arena45.err
timeout 900 $TR --nproc-per-node 4 --master-port 29704 tools/edm_bench.py --layers 32 --dedup-early > $O/edm_n4_L32_dedup_early.json 2> $O/edm1.err
timeout 900 $TR --nproc-per-node 4 --master-port 29705 tools/edm_bench.py --layers 32 > $O/edm_n4_L32.json 2> $O/edm2.err
RS_REMOTE_KERNEL=bulk timeout 600 ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvltx__bytes_data_protocol.sum \
  --clock-control none -k regex:tiles --csv --log-file $O/ncu_p2p_bulk.csv python tools/p2p_profile.py --layers 4 --reps 1 > $O/ncu_p2p_bulk.out 2>&1
RS_REMOTE_KERNEL=bulk timeout 300 python tools/p2p_profile.py --layers 4 --reps 3 > $O/p2p_bulk.json 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=10 > $O/pytest_gpu.txt 2>&1; echo rc=$? >> $O/pytest_gpu.txt
