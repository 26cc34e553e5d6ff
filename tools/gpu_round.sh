#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, then ncu (launch list + full capture of the top kernel).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
if [ "$1" == "ncu" ]; then
  CMD="python bench.py --steps 3 --warmup 3 --points asym2_10b,full --no-cpu-baseline"
  timeout 300 $CMD > gpurun_out/ncu_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:pc_.*_kernel -s 3 -c 1 -o gpurun_out/prof_asym2 $CMD > gpurun_out/ncu_full.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu_full.log
fi
