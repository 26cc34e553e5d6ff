mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02/pytest_fe.log 2>&1; echo "rc=$?" >> gpurun_out/r02/pytest_fe.log
timeout 300 python bench.py --no-sub --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/r02/bench_fe.json 2>&1
timeout 300 python bench.py --workload cfg5 --points adapt_40db,full --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/r02/cfg5_fe.json 2>&1
python tools/tiled_timeline.py cfg2 > gpurun_out/r02/tl_fe.json 2>&1
