mkdir -p gpurun_out/r02
P=gpurun_out/r02
timeout 600 python -m pytest tests -m gpu -q -k "fft" > $P/pytest_fft4.log 2>&1; echo "rc=$?" >> $P/pytest_fft4.log
timeout 300 python bench.py --workload cfg3 --points asym2_q191_fft,asym2_9b_fft,full_fft32k,full_fft --steps 20 --warmup 5 --no-cpu-baseline > $P/bench_cfg3_tw.json 2>&1
python tools/fft_timeline.py 16777216 4096 > $P/fft_tl_tw.json 2>&1
C5="python bench.py --workload cfg5 --L 16777216 --no-cpu-baseline --steps 3 --warmup 3 --points adapt_40db"
CH="python bench.py --no-sub --no-cpu-baseline --steps 20 --warmup 5 --points asym2_10b"
$C5 > $P/plain_5b.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:pc_tiled_kernel<2" -s 3 -c 1 -o $P/prof_cfg5_asym2 $C5 > $P/ncu_5b.log 2>&1
$CH > $P/plain_h.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $P/launches_headline.csv $CH > $P/ncu_h.log 2>&1
echo done
