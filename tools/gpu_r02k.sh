mkdir -p gpurun_out/r02
timeout 300 python bench.py --no-sub --no-cpu-baseline --steps 20 --warmup 5 --points asym2_10b,sym_8b,full > gpurun_out/r02/ef0.json 2>&1
timeout 300 python bench.py --no-sub --no-cpu-baseline --steps 20 --warmup 5 --points asym2_10b,sym_8b,full --opt early_fill=1 > gpurun_out/r02/ef1.json 2>&1
timeout 300 python bench.py --no-sub --no-cpu-baseline --steps 20 --warmup 5 --points asym2_10b,sym_8b,full --graph 0 > gpurun_out/r02/ef0_nog.json 2>&1
timeout 300 python bench.py --no-sub --no-cpu-baseline --steps 20 --warmup 5 --points asym2_10b,sym_8b,full --graph 0 --opt early_fill=1 > gpurun_out/r02/ef1_nog.json 2>&1
