mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests -m gpu -q -x -k "not full_size" > gpurun_out/r02/pytest_a.log 2>&1; echo "rc=$?" >> gpurun_out/r02/pytest_a.log
timeout 600 python -m pytest tests -m gpu -q -k "backend_validation or debug_max or binding_rejects or many_blocks or sharding" -s > gpurun_out/r02/pytest_new.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --points asym2_10b,full --no-cpu-baseline > gpurun_out/r02/bench_cfg2.json 2> gpurun_out/r02/bench_cfg2.err
