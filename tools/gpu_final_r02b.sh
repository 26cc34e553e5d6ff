# Round-2 final GPU pass (after the producer study): every GPU test, smoke, the driver's bench
# command, every workload's bench line, the torchrun launch path (1 rank), the reference arm, the
# core-variant cross-checks for sym/asym3, the headline launch list and ncu summaries.
P=gpurun_out/r02bf
mkdir -p $P
python -c "import __graft_entry__ as g; g.build()" > $P/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > $P/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $P/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $P/smoke.log 2>&1; echo "smoke rc=$?" >> $P/smoke.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $P/bench_default.json 2> $P/bench_default.err
for w in cfg1 cfg3 cfg5; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > $P/bench_$w.json 2> $P/bench_$w.err
done
timeout 900 python bench.py --workload cfg4 --steps 5 --warmup 3 > $P/bench_cfg4.json 2> $P/bench_cfg4.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline --no-sub > $P/bench_torchrun.json 2> $P/bench_torchrun.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > $P/bench_reference.json 2> $P/bench_reference.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-sub --points sym_8b,asym3_8b --opt core_variant=2 > $P/bench_dmma_core.json 2> $P/bench_dmma_core.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-sub --points sym_8b,asym3_8b --opt core_variant=1 > $P/bench_fma_core.json 2> $P/bench_fma_core.err
timeout 300 python tools/tiled_timeline.py cfg2 > $P/timeline_cfg2.json 2> $P/timeline.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $P/launches_headline.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sub --points asym2_10b > $P/ncu_launch.log 2>&1
for pt in asym2_10b sym_8b; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:pc_tiled_kernel -s 4 -c 1 -o $P/prof_cfg2_$pt python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-sub --points $pt > $P/ncu_$pt.log 2>&1
done
echo done
