mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests -m gpu -q -k "randomized or c_example" > gpurun_out/r02/pytest_rand.log 2>&1; echo "rc=$?" >> gpurun_out/r02/pytest_rand.log
