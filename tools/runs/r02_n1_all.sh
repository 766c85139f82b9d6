#!/bin/bash
# Round-2 one-GPU validation + profile (gpurun, 1 GPU): outputs under gpurun_out/r02f/.
O=gpurun_out/r02f; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=10 > $O/pytest_gpu.txt 2>&1; echo rc=$? >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo rc=$? >> $O/smoke.txt
RS_TIMING=1 timeout 900 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err
timeout 900 python bench.py --impl reference > $O/ref_n1.json 2> $O/ref_n1.err
bash tools/runs/r02_n1_profile.sh
