#!/bin/bash
mkdir -p gpurun_out
timeout 200 python bench.py --no-cpu-baseline --points asym2_10b,full --opt 1=16 > gpurun_out/e_T16.json 2>/dev/null
timeout 200 python bench.py --no-cpu-baseline --points asym2_10b,full --opt 1=12 > gpurun_out/e_T12.json 2>/dev/null
timeout 200 python bench.py --no-cpu-baseline --points asym2_10b,full --opt 3=2 > gpurun_out/e_np2.json 2>/dev/null
timeout 200 python bench.py --no-cpu-baseline --points asym2_10b,full --opt 3=1 > gpurun_out/e_np1.json 2>/dev/null
timeout 200 python bench.py --no-cpu-baseline --points asym2_10b,full > gpurun_out/e_base.json 2>/dev/null
