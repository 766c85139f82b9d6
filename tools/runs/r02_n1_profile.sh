#!/bin/bash
# Round-2 one-GPU profile: DRAM traffic of every copy launch of the bench (ncu metrics),
# then one full ncu capture of a forward bulk launch. Outputs under gpurun_out/r02f/.
O=gpurun_out/r02f; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:'bulk_tiles|copy_tiles' --csv --log-file $O/traffic_n1_L32.csv $CMD > $O/ncu_traffic.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:bulk_tiles -s 8 -c 1 -o $O/prof_bulk_n1 $CMD > $O/ncu_full.log 2>&1
ncu -i $O/prof_bulk_n1.ncu-rep --page raw --csv > $O/prof_bulk_n1_raw.csv 2>&1
