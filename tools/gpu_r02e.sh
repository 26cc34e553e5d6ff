mkdir -p gpurun_out/r02
python tools/fft_timeline.py 4194304 4096 5120 8192 > gpurun_out/r02/fft_tl.json 2>&1
PC_LIB_PATH=tools/variants/libpc_minb1.so python tools/fft_timeline.py 4194304 5120 6144 > gpurun_out/r02/fft_tl_minb1.json 2>&1
