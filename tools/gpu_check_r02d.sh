# Re-entry sanity pass after the container re-creation: GPU tests, smoke, the driver's default bench line.
P=gpurun_out/r02d
mkdir -p $P
timeout 900 python -m pytest tests -m gpu -q -x > $P/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $P/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $P/smoke.log 2>&1; echo "smoke rc=$?" >> $P/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > $P/bench_default.json 2> $P/bench_default.err
echo done
