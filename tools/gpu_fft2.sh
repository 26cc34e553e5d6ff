#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -k "fft" > gpurun_out/pt_fft.log 2>&1
for n in 4096 8192; do
timeout 300 python bench.py --workload cfg3 --steps 5 --warmup 2 --no-cpu-baseline --points asym2_9b_fft,full_fft --opt 4=$n > gpurun_out/fftA_$n.json 2> gpurun_out/fftA_$n.err
done
PC_NVCC_EXTRA=-DPC_FFT_TW_AFTER python -c "import __graft_entry__ as g; g.build()" > gpurun_out/buildB.log 2>&1
for n in 4096 8192; do
timeout 300 python bench.py --workload cfg3 --steps 5 --warmup 2 --no-cpu-baseline --points asym2_9b_fft,full_fft --opt 4=$n > gpurun_out/fftB_$n.json 2> gpurun_out/fftB_$n.err
done
