mkdir -p gpurun_out/r02
timeout 300 python bench.py --no-sub --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/r02/bench_pf.json 2>&1
PC_LIB_PATH=tools/variants/pf0.so timeout 300 python bench.py --no-sub --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/r02/bench_pf0.json 2>&1
python tools/tiled_timeline.py cfg2 > gpurun_out/r02/tl_pf.json 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02/pytest_pf.log 2>&1; echo "rc=$?" >> gpurun_out/r02/pytest_pf.log
