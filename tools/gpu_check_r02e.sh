# After the per-block kernel thread change: every GPU test, smoke, cfg1 and default bench lines.
P=gpurun_out/r02e
mkdir -p $P
timeout 900 python -m pytest tests -m gpu -q > $P/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $P/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $P/smoke.log 2>&1; echo "smoke rc=$?" >> $P/smoke.log
for r in 1 2; do timeout 300 python bench.py --workload cfg1 --steps 50 --warmup 5 --no-cpu-baseline > $P/bench_cfg1_$r.json 2> $P/bench_cfg1_$r.err; done
timeout 600 python bench.py --steps 20 --warmup 5 > $P/bench_default.json 2> $P/bench_default.err
echo done
