#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tools/tiled_timeline.py cfg2 > gpurun_out/tl_cfg2.json 2> gpurun_out/tl_cfg2.err
