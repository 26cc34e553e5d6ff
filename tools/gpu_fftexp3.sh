#!/bin/bash
mkdir -p gpurun_out
for c in 60 70 100; do
PC_NVCC_EXTRA="-DPC_FFT_CARVEOUT=$c" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bC$c.log 2>&1
timeout 200 python tools/fft_timeline.py > gpurun_out/fft_tl_c$c.json 2> gpurun_out/fft_tl_c$c.err
timeout 300 python bench.py --workload cfg3 --steps 5 --warmup 2 --no-cpu-baseline --points asym2_9b_fft,full_fft > gpurun_out/fft_c$c.json 2>gpurun_out/fft_c$c.err
done
