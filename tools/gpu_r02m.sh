mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02/pytest_m.log 2>&1; echo "rc=$?" >> gpurun_out/r02/pytest_m.log
timeout 300 python bench.py --workload cfg5 --points adapt_40db,full --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/r02/cfg5_m.json 2>&1
