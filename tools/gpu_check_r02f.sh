# Re-entry pass on the rebuilt library: every GPU test, smoke, the default bench line, its ncu launch list.
P=gpurun_out/r02f
mkdir -p $P
timeout 900 python -m pytest tests -m gpu -q > $P/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $P/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $P/smoke.log 2>&1; echo "smoke rc=$?" >> $P/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > $P/bench_default.json 2> $P/bench_default.err; echo "bench rc=$?" >> $P/bench_default.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $P/launches_headline.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $P/ncu_bench.log 2>&1
echo done
