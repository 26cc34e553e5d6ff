mkdir -p gpurun_out/r02
for lib in paper_1201_3018_b200/libpackedconv.so tools/variants/h1.so tools/variants/h2.so tools/variants/h3.so tools/variants/h4.so; do
  PC_LIB_PATH=$lib python tools/e2e_check.py pg > gpurun_out/r02/e2e_$(basename $lib .so).log 2>&1
done
python tools/pcie_probe.py > gpurun_out/r02/pcie2.log 2>&1
