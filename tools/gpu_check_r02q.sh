# Last pass of round 2 on HEAD (default build): every GPU test, smoke, default bench line, launch list, cfg1 line, cfg2 points.
P=gpurun_out/r02q
mkdir -p $P
timeout 900 python -m pytest tests -m gpu -q > $P/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $P/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $P/smoke.log 2>&1; echo "smoke rc=$?" >> $P/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > $P/bench_default.json 2> $P/bench_default.err; echo "bench rc=$?" >> $P/bench_default.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $P/launches_headline.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $P/ncu_bench.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/round_check0 tools/round_check.cu > /dev/null 2>&1 && /tmp/round_check0 > $P/round_check_default.log 2>&1
timeout 300 python bench.py --workload cfg1 --steps 50 --warmup 5 --no-cpu-baseline > $P/bench_cfg1.json 2> $P/bench_cfg1.err
timeout 300 python bench.py --no-sub --no-cpu-baseline --steps 20 --warmup 5 --points asym2_10b,asym2_8b,asym3_8b,sym_8b > $P/bench_cfg2_points.json 2> $P/bench_cfg2_points.err
echo done
