#!/bin/bash
mkdir -p gpurun_out
for n in 2048 4096 8192; do
timeout 300 python bench.py --workload cfg3 --steps 5 --warmup 2 --no-cpu-baseline --points asym2_9b_fft,full_fft --opt 4=$n > gpurun_out/fft_$n.json 2> gpurun_out/fft_$n.err
done
