#!/bin/bash
# Round-2 final multi-GPU validation (gpurun --gpus 4): outputs under gpurun_out/r02zm/.
O=gpurun_out/${OUT:-r02zm}; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rs --durations=10 > $O/pytest_gpu.txt 2>&1; echo rc=$? >> $O/pytest_gpu.txt
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node 2 --master-port 29961 bench.py --gpus 2 > $O/bench_n2.json 2> $O/bench_n2.err
timeout 900 $TR --nproc-per-node 4 --master-port 29962 bench.py --gpus 4 > $O/bench_n4.json 2> $O/bench_n4.err
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err
timeout 900 $TR --nproc-per-node 4 --master-port 29963 bench.py --impl reference --gpus 4 > $O/ref_n4.json 2> $O/ref_n4.err
