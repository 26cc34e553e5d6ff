# A/B of the add-based companding rounding (PC_RND_ADD=1; in-tree build = the variant): the
# rounding checker, every GPU test, cfg2 points, cfg3 FFT and cfg1 lines, timelines.
P=gpurun_out/r02i_rint; mkdir -p $P
./tools/round_check > $P/round_check.log 2>&1; echo "rc=$?" >> $P/round_check.log
SKIP_TESTS= bash tools/gpu_ab.sh r02i_rint "base rint2" asym2_10b,sym_8b,asym3_8b 3
for r in 1 2; do for v in base rint2; do
  PC_LIB_PATH=$PWD/tools/variants/$v.so timeout 300 python bench.py --workload cfg3 --steps 10 --warmup 3 --no-cpu-baseline --points asym2_q191_fft > $P/cfg3_${v}_$r.json 2> $P/cfg3_${v}_$r.err
  PC_LIB_PATH=$PWD/tools/variants/$v.so timeout 300 python bench.py --workload cfg1 --steps 50 --warmup 5 --no-cpu-baseline > $P/cfg1_${v}_$r.json 2> $P/cfg1_${v}_$r.err
done; done
echo done
