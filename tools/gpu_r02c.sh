mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests -m gpu -q -k "host_blocks or adapt_blocks or best_match" > gpurun_out/r02/pytest_c.log 2>&1; echo "rc=$?" >> gpurun_out/r02/pytest_c.log
python tools/e2e_check.py > gpurun_out/r02/e2e_check.log 2>&1
python tools/e2e_check.py pg >> gpurun_out/r02/e2e_check.log 2>&1
