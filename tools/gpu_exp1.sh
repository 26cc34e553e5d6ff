#!/bin/bash
mkdir -p gpurun_out
python tools/tiled_timeline.py cfg2 > gpurun_out/tl_cfg2.json 2> gpurun_out/tl_cfg2.err
for c in 1 2 3 4; do for T in 14 16; do
python bench.py --points asym2_10b,full --no-cpu-baseline --steps 30 --opt 2=$c --opt 1=$T > gpurun_out/exp_c${c}_T$T.json 2>/dev/null
done; done
python bench.py --L 16777216 --points asym2_10b,full --no-cpu-baseline --steps 20 > gpurun_out/exp_L24.json 2>/dev/null
