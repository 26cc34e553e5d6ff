mkdir -p gpurun_out/r02
P=gpurun_out/r02
C5="python bench.py --workload cfg5 --L 16777216 --no-cpu-baseline --steps 3 --warmup 3 --points adapt_40db"
$C5 > $P/plain_5c.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:pc_tiled_kernel<\(int\)2' -s 3 -c 1 -o $P/prof_cfg5_asym2 $C5 > $P/ncu_5c.log 2>&1
echo done
