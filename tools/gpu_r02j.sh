mkdir -p gpurun_out/r02
for lib in paper_1201_3018_b200/libpackedconv.so tools/variants/v1_s1_pk.so tools/variants/v2_s1_nopk.so tools/variants/v3_s2_nopk.so; do
  n=$(basename $lib .so)
  PC_LIB_PATH=$lib timeout 300 python bench.py --no-sub --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/r02/sl_$n.json 2>&1
  PC_LIB_PATH=$lib python tools/tiled_timeline.py cfg2 > gpurun_out/r02/tl_sl_$n.json 2>&1
done
