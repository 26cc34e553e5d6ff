# Round-2 profile pass: ncu --set full of the hot kernels (each command first run plain, then under ncu)
# and the launch list of the default bench command.
mkdir -p gpurun_out/r02
P=gpurun_out/r02
C2A="python bench.py --no-sub --no-cpu-baseline --steps 3 --warmup 3 --points asym2_10b"
C2F="python bench.py --no-sub --no-cpu-baseline --steps 3 --warmup 3 --points full"
C2S="python bench.py --no-sub --no-cpu-baseline --steps 3 --warmup 3 --points sym_8b"
C3="python bench.py --workload cfg3 --no-cpu-baseline --steps 3 --warmup 3 --points asym2_q191_fft"
C5="python bench.py --workload cfg5 --L 16777216 --no-cpu-baseline --steps 3 --warmup 3 --points adapt_40db"
CD="python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
$C2A > $P/plain_a.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:pc_tiled_kernel -s 3 -c 1 -o $P/prof_cfg2_asym2 $C2A > $P/ncu_a.log 2>&1
$C2F > $P/plain_f.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:pc_tiled_kernel -s 3 -c 1 -o $P/prof_cfg2_full $C2F > $P/ncu_f.log 2>&1
$C2S > $P/plain_s.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:pc_tiled_kernel -s 3 -c 1 -o $P/prof_cfg2_sym $C2S > $P/ncu_s.log 2>&1
$C3 > $P/plain_3.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:pc_fft_conv -s 3 -c 1 -o $P/prof_cfg3_fft $C3 > $P/ncu_3.log 2>&1
$C5 > $P/plain_5.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k "regex:pc_tiled_kernel<2" -s 3 -c 1 -o $P/prof_cfg5_asym2 $C5 > $P/ncu_5.log 2>&1
$CD > $P/plain_d.log 2>&1 && timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $P/launches_default.csv $CD > $P/ncu_d.log 2>&1
echo done
