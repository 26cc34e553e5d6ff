# A/B of library variants (tools/variants/<name>.so via PC_LIB_PATH): GPU tests on the in-tree
# build, then alternating cfg2 bench runs of each variant, then a timeline per variant.
# usage: bash tools/gpu_ab.sh OUTDIR "base v1" [points] [reps] [extra bench args]
P=gpurun_out/$1; V=$2; PTS=${3:-asym2_10b,sym_8b}; REPS=${4:-3}; EXTRA=$5
mkdir -p $P
if [ -z "$SKIP_TESTS" ]; then
timeout 900 python -m pytest tests -m gpu -q -x > $P/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $P/pytest_gpu.log
fi
for r in $(seq 1 $REPS); do
  for v in $V; do
    PC_LIB_PATH=$PWD/tools/variants/$v.so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-sub --points $PTS $EXTRA > $P/bench_${v}_$r.json 2> $P/bench_${v}_$r.err
  done
done
for v in $V; do
  PC_LIB_PATH=$PWD/tools/variants/$v.so timeout 300 python tools/tiled_timeline.py cfg2 > $P/timeline_$v.json 2> $P/timeline_$v.err
done
echo done
