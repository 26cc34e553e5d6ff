mkdir -p gpurun_out/r02
timeout 600 python -m pytest tests -m gpu -q -k "fft or backend" > gpurun_out/r02/pytest_cl.log 2>&1; echo "rc=$?" >> gpurun_out/r02/pytest_cl.log
timeout 300 python bench.py --workload cfg3 --points asym2_q191_fft,asym2_9b_fft,full_fft32k,full_fft --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02/bench_cfg3_cl.json 2>&1
python tools/fft_timeline.py 16777216 4096 > gpurun_out/r02/fft_tl_cl.json 2>&1
