# A/B of library variants on the cfg1 line (bench.py --workload cfg1): $1 out dir, $2 variants, $3 reps
P=gpurun_out/$1; mkdir -p $P
for r in $(seq 1 ${3:-2}); do
  for v in $2; do
    PC_LIB_PATH=$PWD/tools/variants/$v.so timeout 300 python bench.py --workload cfg1 --steps 50 --warmup 5 --no-cpu-baseline > $P/bench_${v}_$r.json 2> $P/bench_${v}_$r.err
  done
done
echo done
