#!/bin/bash
# Round-2 multi-GPU batch 3 (gpurun --gpus 4): outputs under gpurun_out/r02m3/.
O=gpurun_out/r02m3; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 900 $TR --nproc-per-node 4 --master-port 29801 tools/edm_bench.py --layers 32 --dedup-early > $O/edm_n4_L32_dedup_early.json 2> $O/edm1.err
timeout 900 $TR --nproc-per-node 4 --master-port 29802 tools/edm_bench.py --layers 32 > $O/edm_n4_L32.json 2> $O/edm2.err
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR --nproc-per-node 2 --master-port 29803 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_n2.json 2> $O/bench_n2.err
timeout 600 $TR --nproc-per-node 4 --master-port 29804 bench.py --gpus 4 --steps 5 --warmup 3 --no-cpu-baseline --transport nccl > $O/bench_n4_nccl.json 2> $O/bench_n4_nccl.err
timeout 900 $TR --nproc-per-node 4 --master-port 29805 tools/configs_bench.py --config 1 --config 4 --config 3 --reps 3 > $O/configs_n4.jsonl 2> $O/configs.err
timeout 900 $TR --nproc-per-node 4 --master-port 29806 tools/configs_bench.py --config 4 --layers 48 --arena-cap 170 --reps 2 > $O/config4_full_n4_cap170.json 2> $O/config4.err
timeout 900 $TR --nproc-per-node 4 --master-port 29807 tools/configs_bench.py --config 5 --layers 40 --arena-cap 180 --reps 3 --host-barriers > $O/config5_n4_L40_cap180_host.json 2> $O/config5h.err
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=10 > $O/pytest_gpu.txt 2>&1; echo rc=$? >> $O/pytest_gpu.txt
