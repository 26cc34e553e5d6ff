mkdir -p gpurun_out/r02
for lib in paper_1201_3018_b200/libpackedconv.so tools/variants/libpc_fill4.so; do
  PC_LIB_PATH=$lib timeout 300 python bench.py --no-sub --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/r02/fill_$(basename $lib .so).json 2>&1
  PC_LIB_PATH=$lib timeout 300 python bench.py --workload cfg5 --points adapt_40db,full --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/r02/fill5_$(basename $lib .so).json 2>&1
done
timeout 600 python -m pytest tests -m gpu -q -x -k "not full_size" > gpurun_out/r02/pytest_fill.log 2>&1; echo "rc=$?" >> gpurun_out/r02/pytest_fill.log
