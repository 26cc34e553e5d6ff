mkdir -p gpurun_out
for w in 2 3 4; do python bench.py --points asym2_10b,sym_8b,full --no-cpu-baseline --force-warps $w > gpurun_out/warps_$w.json 2>&1; done
