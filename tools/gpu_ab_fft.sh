# A/B of library variants on the cfg3 FFT line (bench.py --workload cfg3)
P=gpurun_out/$1; mkdir -p $P
for r in $(seq 1 ${3:-2}); do
  for v in $2; do
    PC_LIB_PATH=$PWD/tools/variants/$v.so timeout 300 python bench.py --workload cfg3 --steps 10 --warmup 3 --no-cpu-baseline --points ${4:-asym2_q191_fft,full_fft} > $P/bench_${v}_$r.json 2> $P/bench_${v}_$r.err
  done
done
echo done
