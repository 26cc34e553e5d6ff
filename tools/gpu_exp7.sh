#!/bin/bash
mkdir -p gpurun_out
for N in 128 256; do for ex in perblock fused; do
timeout 200 python bench.py --workload cfg1 --N $N --L 1048576 --steps 100 --no-cpu-baseline --exec $ex --points asym2_8b,sym_q44,full > gpurun_out/y_${N}_$ex.json 2>gpurun_out/y_${N}_$ex.err
done; done
for N in 128 256; do for ex in perblock fused; do
timeout 200 python bench.py --workload cfg2 --N $N --steps 30 --no-cpu-baseline --exec $ex --points asym2_10b,sym_8b,full > gpurun_out/z_${N}_$ex.json 2>gpurun_out/z_${N}_$ex.err
done; done
