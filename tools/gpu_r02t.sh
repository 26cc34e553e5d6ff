mkdir -p gpurun_out/r02
for v in st6 st12; do
PC_LIB_PATH=tools/variants/$v.so timeout 300 python bench.py --workload cfg3 --points asym2_q191_fft,full_fft --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02/bench_cfg3_$v.json 2>&1
PC_LIB_PATH=tools/variants/$v.so python tools/fft_timeline.py 16777216 4096 > gpurun_out/r02/fft_tl_$v.json 2>&1
done
