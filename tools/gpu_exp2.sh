#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tools/tiled_timeline.py cfg2 2120544 > gpurun_out/tl_cfg2_4jobs.json 2> gpurun_out/tl_e1.err
timeout 120 python tools/tiled_timeline.py cfg2 4241088 > gpurun_out/tl_cfg2_8jobs.json 2> gpurun_out/tl_e2.err
timeout 300 python bench.py --workload cfg1 --steps 200 --no-cpu-baseline > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
