# Post-twiddle-padding pass: every GPU test, smoke, the default bench line and the cfg3 line.
P=gpurun_out/r02cf
mkdir -p $P
timeout 900 python -m pytest tests -m gpu -q > $P/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $P/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $P/smoke.log 2>&1; echo "smoke rc=$?" >> $P/smoke.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $P/bench_default.json 2> $P/bench_default.err
timeout 600 python bench.py --workload cfg3 --steps 20 --warmup 5 --no-cpu-baseline > $P/bench_cfg3.json 2> $P/bench_cfg3.err
echo done
