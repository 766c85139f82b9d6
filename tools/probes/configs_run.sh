# BASELINE configs 1, 3, 4, 5 through the fused executor (tools/configs_bench.py)
N=${1:-4}
run() { if [ $N -gt 1 ]; then timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2957$N tools/configs_bench.py "$@"; else timeout 900 python tools/configs_bench.py "$@"; fi; }
if [ $N -gt 1 ]; then
  run --config 1 --config 3 2>/dev/null | grep "^{"
  run --config 4 --layers 24 2>/dev/null | grep "^{"
  run --config 5 --layers 16 2>/dev/null | grep "^{"
else
  run --config 1 2>/dev/null | grep "^{"
  run --config 4 --layers 8 2>/dev/null | grep "^{"
  run --config 5 --layers 4 2>/dev/null | grep "^{"
fi
