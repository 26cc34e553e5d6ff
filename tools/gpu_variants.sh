mkdir -p gpurun_out/r02
P=gpurun_out/r02
C2A="python bench.py --no-sub --no-cpu-baseline --steps 3 --warmup 3 --points asym2_10b"
$C2A > $P/plain_a2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:pc_tiled_kernel -s 3 -c 1 -o $P/prof_cfg2_asym2_fe $C2A > $P/ncu_a2.log 2>&1
CH="python bench.py --no-sub --no-cpu-baseline --steps 20 --warmup 5 --points asym2_10b"
$CH > $P/plain_h2.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $P/launches_headline2.csv $CH > $P/ncu_h2.log 2>&1
echo done
