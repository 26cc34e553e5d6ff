# Round-2 profile pass: ncu --set full of the hot kernels (each command first run plain, then under ncu),
# summarised on the box by tools/ncu_summary.py (gpurun brings back <= 64 MiB: only the headline
# report itself travels back) and the launch list of the default bench command.
mkdir -p gpurun_out/r02p
P=gpurun_out/r02p
C2A="python bench.py --no-sub --no-cpu-baseline --steps 3 --warmup 3 --points asym2_10b"
C2F="python bench.py --no-sub --no-cpu-baseline --steps 3 --warmup 3 --points full"
C2S="python bench.py --no-sub --no-cpu-baseline --steps 3 --warmup 3 --points sym_8b"
C3="python bench.py --workload cfg3 --no-cpu-baseline --steps 3 --warmup 3 --points asym2_q191_fft"
C5="python bench.py --workload cfg5 --L 16777216 --no-cpu-baseline --steps 3 --warmup 3 --points adapt_40db"
CD="python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
prof() {  # name cmd kernel-regex (demangled names: the template arguments read "(int)2")
  $2 > $P/plain_$1.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$3" -s 3 -c 1 -o $P/prof_$1 $2 > $P/ncu_$1.log 2>&1
  python tools/ncu_summary.py $P/prof_$1.ncu-rep $P/ncu_$1.json > /dev/null 2>&1
}
prof cfg2_asym2 "$C2A" regex:pc_tiled_kernel
prof cfg2_full "$C2F" regex:pc_tiled_kernel
prof cfg2_sym "$C2S" regex:pc_tiled_kernel
prof cfg3_fft "$C3" regex:pc_fft_conv
prof cfg5_asym2 "$C5" 'regex:pc_tiled_kernel<\(int\)2'
for n in cfg2_full cfg2_sym cfg3_fft cfg5_asym2; do rm -f $P/prof_$n.ncu-rep; done
$CD > $P/plain_d.log 2>&1 && timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $P/launches_default.csv $CD > $P/ncu_d.log 2>&1
echo done
