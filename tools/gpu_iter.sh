#!/bin/bash
# quick iteration: GPU parity tests + timeline + cfg2 bench (every step under its own timeout)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 120 python tools/tiled_timeline.py cfg2 > gpurun_out/tl_cfg2.json 2> gpurun_out/tl_cfg2.err
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
