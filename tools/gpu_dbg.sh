#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tools/dbg_tiled.py 1000 9 40 2 7 > gpurun_out/dbg1.log 2>&1; echo "rc=$?" >> gpurun_out/dbg1.log
timeout 120 python tools/dbg_tiled.py 1000 9 40 1 7 > gpurun_out/dbg2.log 2>&1; echo "rc=$?" >> gpurun_out/dbg2.log
timeout 120 python tools/dbg_tiled.py 4194304 512 4096 2 511 > gpurun_out/dbg3.log 2>&1; echo "rc=$?" >> gpurun_out/dbg3.log
timeout 120 python tools/dbg_tiled.py 4194304 512 4096 0 0 > gpurun_out/dbg4.log 2>&1; echo "rc=$?" >> gpurun_out/dbg4.log
timeout 120 python tools/dbg_tiled.py 4194304 512 4096 1 127 > gpurun_out/dbg5.log 2>&1; echo "rc=$?" >> gpurun_out/dbg5.log
