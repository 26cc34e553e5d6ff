nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/peak_clocks.csv &
SMI=$!
mkdir -p gpurun_out; ./tools/fp64_peak > gpurun_out/fp64_peak.log 2>&1
kill $SMI
nvidia-smi -q | grep -i -A3 "clocks" | head -40 >> gpurun_out/fp64_peak.log
nproc >> gpurun_out/fp64_peak.log; lscpu | head -20 >> gpurun_out/fp64_peak.log
