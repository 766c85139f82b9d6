#!/bin/bash
# NVLink push knob sweep, 2 GPUs from one process (tools/p2p_profile.py, L=8)
O=gpurun_out/r02sw; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
for v in 1 0; do for c in 1 2 3 4; do for t in 262144 524288 1048576 2097152; do
  RS_VEC32=$v timeout 120 python tools/p2p_profile.py --layers 8 --reps 3 --ctas $c --tile-bytes $t 2>/dev/null | tail -1 | sed "s/^/vec32=$v /" >> $O/sweep.txt
done; done; done
