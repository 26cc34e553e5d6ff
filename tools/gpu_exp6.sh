#!/bin/bash
mkdir -p gpurun_out
for L in 131072 262144 524288 1048576; do
for ex in perblock fused; do
timeout 200 python bench.py --workload cfg1 --L $L --steps 100 --no-cpu-baseline --exec $ex --points asym2_9b,full > gpurun_out/x_${L}_$ex.json 2>/dev/null
done; done
