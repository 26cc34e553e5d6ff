mkdir -p gpurun_out/r02
PC_LIB_PATH=tools/variants/fft3.so timeout 300 python bench.py --workload cfg3 --points asym2_q191_fft,full_fft --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02/bench_cfg3_m3.json 2>&1
PC_LIB_PATH=tools/variants/fft3.so python tools/fft_timeline.py 16777216 4096 > gpurun_out/r02/fft_tl_m3.json 2>&1
