mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02/pytest_b.log 2>&1; echo "rc=$?" >> gpurun_out/r02/pytest_b.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02/bench_default.json 2> gpurun_out/r02/bench_default.err; echo "rc=$?" >> gpurun_out/r02/bench_default.err
