mkdir -p gpurun_out/r02
for v in f6 f8 s3; do
PC_LIB_PATH=tools/variants/$v.so timeout 300 python bench.py --no-sub --no-cpu-baseline --steps 20 --warmup 5 --points asym2_10b,asym3_8b,full > gpurun_out/r02/bench_v2_$v.json 2>&1
done
timeout 300 python bench.py --no-sub --no-cpu-baseline --steps 20 --warmup 5 --points asym2_10b,asym3_8b,full > gpurun_out/r02/bench_v2_base.json 2>&1
