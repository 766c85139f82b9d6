#!/bin/bash
# Round-2 multi-GPU measurement batch (run under gpurun --gpus 4). Every step has its own
# timeout; outputs under gpurun_out/r02m/.
O=gpurun_out/r02m; mkdir -p $O
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
# 1. bench N=2 / N=4, 256-bit vectors on (default) and off
for n in 2 4; do
  [ $N -ge $n ] || continue
  for v in 1 0; do
    RS_VEC32=$v timeout 600 $TR --nproc-per-node $n --master-port $((29600+n*10+v)) bench.py --gpus $n --steps 5 --warmup 3 --no-cpu-baseline \
      > $O/bench_n${n}_vec32_$v.json 2> $O/bench_n${n}_vec32_$v.err
  done
done
# 2. ncu NVLink protocol bytes of the peer push, 2 GPUs from one process, vec32 on / off
for v in 1 0; do
  RS_VEC32=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvltx__bytes_data_protocol.sum,nvlrx__bytes.sum \
    --clock-control none -k regex:tiles --csv --log-file $O/ncu_p2p_vec32_$v.csv python tools/p2p_profile.py --layers 4 --reps 1 > $O/ncu_p2p_vec32_$v.out 2>&1
  RS_VEC32=$v timeout 300 python tools/p2p_profile.py --layers 4 --reps 3 > $O/p2p_vec32_$v.json 2>&1
done
# 3. config 5 at N=4, L=40 (the per-GPU state of the full model at N=8) under 180 GB, device vs host stage barriers
if [ $N -ge 4 ]; then
  timeout 900 $TR --nproc-per-node 4 --master-port 29651 tools/configs_bench.py --config 5 --layers 40 --arena-cap 180 --reps 2 > $O/config5_n4_L40_cap180_device.json 2> $O/config5_dev.err
  timeout 900 $TR --nproc-per-node 4 --master-port 29652 tools/configs_bench.py --config 5 --layers 40 --arena-cap 180 --reps 2 --host-barriers > $O/config5_n4_L40_cap180_host.json 2> $O/config5_host.err
  # 4. north star under a per-GPU cap at N=4: many memory-aware stages with device barriers vs no arena
  timeout 600 $TR --nproc-per-node 4 --master-port 29653 bench.py --gpus 4 --steps 5 --warmup 3 --no-cpu-baseline --arena-multi --hbm-cap 45000000000 > $O/bench_n4_arena45.json 2> $O/bench_n4_arena45.err
  timeout 600 $TR --nproc-per-node 4 --master-port 29654 bench.py --gpus 4 --steps 5 --warmup 3 --no-cpu-baseline --arena-multi > $O/bench_n4_arena_free.json 2> $O/bench_n4_arena_free.err
fi
# 5. the GPU test suite on this box
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=10 > $O/pytest_gpu.txt 2>&1; echo rc=$? >> $O/pytest_gpu.txt
