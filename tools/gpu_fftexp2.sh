#!/bin/bash
mkdir -p gpurun_out
PC_NVCC_EXTRA="-DPC_FFT_NOTW" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bN.log 2>&1
timeout 200 python tools/fft_timeline.py > gpurun_out/fft_tl_notw.json 2> gpurun_out/fft_tl_notw.err
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bN2.log 2>&1
timeout 200 python tools/fft_timeline.py > gpurun_out/fft_tl.json 2> gpurun_out/fft_tl.err
