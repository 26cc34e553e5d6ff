# Final profile pass of round 2: ncu --set full of the headline tiled kernel and of the per-block
# kernel (cfg1, after the >= 256-thread change); each command first exits 0 without ncu.
mkdir -p gpurun_out/r02kp
P=gpurun_out/r02kp
C2A="python bench.py --no-sub --no-cpu-baseline --steps 3 --warmup 3 --points asym2_10b"
C1="python bench.py --workload cfg1 --no-cpu-baseline --steps 3 --warmup 3 --points asym2_9b"
prof() {
  $2 > $P/plain_$1.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$3" -s 3 -c 1 -o $P/prof_$1 $2 > $P/ncu_$1.log 2>&1
  python tools/ncu_summary.py $P/prof_$1.ncu-rep $P/ncu_$1.json > /dev/null 2>&1
}
prof cfg2_asym2 "$C2A" regex:pc_tiled_kernel
prof cfg1_asym2 "$C1" regex:pc_fused_kernel
rm -f $P/prof_cfg2_asym2.ncu-rep
echo done
