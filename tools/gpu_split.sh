# producer-SM mode sweep (conv_opts.prepack = -P) on cfg2, against the base library
mkdir -p gpurun_out/$1
for P in $2; do
  PC_LIB_PATH=$PWD/tools/variants/$3.so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-sub --points ${4:-asym2_10b} --opt prepack=-$P > gpurun_out/$1/bench_P$P.json 2> gpurun_out/$1/bench_P$P.err
done
PC_LIB_PATH=$PWD/tools/variants/base.so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-sub --points ${4:-asym2_10b} > gpurun_out/$1/bench_base.json 2> gpurun_out/$1/bench_base.err
for P in $5; do
  PC_OPT="prepack=-$P" PC_LIB_PATH=$PWD/tools/variants/$3.so timeout 300 python tools/tiled_timeline.py cfg2 > gpurun_out/$1/tl_P$P.json 2> gpurun_out/$1/tl_P$P.err
done
echo done
