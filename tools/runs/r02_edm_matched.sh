#!/bin/bash
# Config 3 through the EDM at N=4 with the matched placement (gpurun --gpus 4): gpurun_out/r02em/.
O=gpurun_out/r02em; mkdir -p $O
timeout 900 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4 --master-port 29996 \
    tools/edm_bench.py --layers 32 --dedup-early > $O/edm_matched_dedup_early.json 2> $O/edm_matched_dedup_early.err
