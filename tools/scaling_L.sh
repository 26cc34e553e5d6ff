mkdir -p gpurun_out
for L in 1048576 2097152 4194304 8388608 16777216; do
  python bench.py --L $L --points asym2_10b,sym_8b,full --no-cpu-baseline --steps 30 > gpurun_out/scal_$L.json 2>/dev/null
done
