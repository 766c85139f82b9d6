#!/bin/bash
# Round-2 multi-GPU batch 6 (gpurun --gpus 4): the final code at N=2/4. Outputs under gpurun_out/r02m6/.
O=gpurun_out/r02m6; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
CUDA_VISIBLE_DEVICES=0,1 RS_TIMING=1 timeout 600 $TR --nproc-per-node 2 --master-port 29931 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_n2.json 2> $O/bench_n2.err
RS_TIMING=1 timeout 600 $TR --nproc-per-node 4 --master-port 29932 bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_n4.json 2> $O/bench_n4.err
timeout 600 $TR --nproc-per-node 4 --master-port 29933 bench.py --gpus 4 --steps 5 --warmup 3 --no-cpu-baseline --arena-multi --hbm-cap 45000000000 > $O/bench_n4_arena45.json 2> $O/bench_n4_arena45.err
timeout 900 $TR --nproc-per-node 4 --master-port 29934 tools/configs_bench.py --config 5 --layers 40 --arena-cap 180 --reps 3 > $O/config5_n4_L40_cap180.json 2> $O/config5.err
timeout 900 $TR --nproc-per-node 4 --master-port 29935 tools/edm_bench.py --layers 32 --dedup-early > $O/edm_n4_L32_dedup_early.json 2> $O/edm.err
timeout 1800 python -m pytest tests -m gpu -q -rs --durations=10 > $O/pytest_gpu.txt 2>&1; echo rc=$? >> $O/pytest_gpu.txt
