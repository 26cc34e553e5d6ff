#!/bin/bash
mkdir -p gpurun_out
C="python bench.py --steps 3 --warmup 3 --points asym2_10b --no-cpu-baseline"
timeout 300 $C > gpurun_out/ncu_plain.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pc_tiled_kernel -s 3 -c 1 -o gpurun_out/prof_cfg2_asym2 $C > gpurun_out/ncu_full_cfg2.log 2>&1
C="python bench.py --steps 3 --warmup 3 --points full --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pc_tiled_kernel -s 3 -c 1 -o gpurun_out/prof_cfg2_full $C > gpurun_out/ncu_full_cfg2f.log 2>&1
echo done
