#!/bin/bash
# ncu: launch list of the cfg2 bench command + --set full captures of the hot kernels (cfg2 tiled, cfg3 FFT, cfg5 adaptive).
mkdir -p gpurun_out
C2="python bench.py --steps 3 --warmup 3 --points asym2_10b,full --no-cpu-baseline"
timeout 300 $C2 > gpurun_out/ncu_plain.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv $C2 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pc_tiled_kernel -s 3 -c 1 -o gpurun_out/prof_cfg2_asym2 python bench.py --steps 3 --warmup 3 --points asym2_10b --no-cpu-baseline > gpurun_out/ncu_full_cfg2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pc_tiled_kernel -s 3 -c 1 -o gpurun_out/prof_cfg2_full python bench.py --steps 3 --warmup 3 --points full --no-cpu-baseline > gpurun_out/ncu_full_cfg2f.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pc_fft -s 3 -c 1 -o gpurun_out/prof_cfg3_fft python bench.py --workload cfg3 --steps 3 --warmup 3 --points asym2_9b_fft --no-cpu-baseline > gpurun_out/ncu_full_cfg3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pc_fused -s 3 -c 1 -o gpurun_out/prof_cfg5_adapt python bench.py --workload cfg5 --L 16777216 --steps 3 --warmup 3 --points adapt_40db --no-cpu-baseline > gpurun_out/ncu_full_cfg5.log 2>&1
echo done
