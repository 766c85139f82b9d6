# copy-engine offload of large contiguous peer-bound blocks, variants (fused executor, north star)
for n in ${1:-2 4}; do
for v in "RS_CE_MIN_BYTES=0" "RS_CE_MIN_BYTES=4194304 RS_CE_STREAMS=2" "RS_CE_MIN_BYTES=4194304 RS_CE_STREAMS=4" "RS_CE_MIN_BYTES=67108864 RS_CE_STREAMS=4"; do
env $v timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n bench.py --gpus $n --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/cev.log 2>&1
echo "N=$n $v: $(grep '^{' gpurun_out/cev.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["reconfig_s"], d["reconfig_back_s"], d["verified_mismatches"])')"
done; done
