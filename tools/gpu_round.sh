#!/bin/bash
# One gpurun call for a round: GPU parity tests, smoke, every bench line, ncu evidence, timelines, sweep.
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash tools/gpu_round.sh'
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
bash tools/gpu_profile.sh                                   # bench_all + ncu + tiled timeline
timeout 200 python tools/fft_timeline.py > gpurun_out/fft_tl.json 2> gpurun_out/fft_tl.err
timeout 600 python tools/sweep_n.py > gpurun_out/sweep_n.json 2> gpurun_out/sweep_n.err
