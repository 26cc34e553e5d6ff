#!/bin/bash
mkdir -p gpurun_out
for v in "8 4" "16 4" "8 8" "16 8"; do set -- $v
PC_NVCC_EXTRA="-DPC_FFT_PEAK_U=$1 -DPC_FFT_PACK_UB=$2" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bv.log 2>&1
timeout 200 python tools/fft_timeline.py > gpurun_out/fft_tl_$1_$2.json 2>/dev/null
timeout 300 python bench.py --workload cfg3 --steps 5 --warmup 2 --no-cpu-baseline --points asym2_9b_fft,full_fft > gpurun_out/fft_$1_$2.json 2>/dev/null
done
