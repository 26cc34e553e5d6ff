#!/bin/bash
# Round profile pass: all bench lines, launch list of the default bench, ncu --set full of the hot kernels.
mkdir -p gpurun_out
bash tools/bench_all.sh
C2="python bench.py --steps 3 --warmup 3 --points asym2_10b,full --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv $C2 > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pc_tiled_kernel -s 3 -c 1 -o gpurun_out/prof_cfg2_asym2 python bench.py --steps 3 --warmup 3 --points asym2_10b --no-cpu-baseline > gpurun_out/ncu_a.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pc_tiled_kernel -s 3 -c 1 -o gpurun_out/prof_cfg2_full python bench.py --steps 3 --warmup 3 --points full --no-cpu-baseline > gpurun_out/ncu_b.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pc_fft_conv -s 3 -c 1 -o gpurun_out/prof_cfg3_fft python bench.py --workload cfg3 --steps 3 --warmup 3 --points asym2_9b_fft --no-cpu-baseline > gpurun_out/ncu_c.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pc_tiled_kernel -s 3 -c 1 -o gpurun_out/prof_cfg5_adapt python bench.py --workload cfg5 --L 16777216 --steps 3 --warmup 3 --points adapt_40db --no-cpu-baseline > gpurun_out/ncu_d.log 2>&1
timeout 120 python tools/tiled_timeline.py cfg2 > gpurun_out/tl_cfg2.json 2> gpurun_out/tl_cfg2.err
echo done
