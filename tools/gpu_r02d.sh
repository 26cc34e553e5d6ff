mkdir -p gpurun_out/r02
timeout 600 python -m pytest tests -m gpu -q -k "fft" > gpurun_out/r02/pytest_fft.log 2>&1; echo "rc=$?" >> gpurun_out/r02/pytest_fft.log
for lib in paper_1201_3018_b200/libpackedconv.so tools/variants/libpc_minb1.so; do
  for n in 4096 5120 6144 8192; do
    PC_LIB_PATH=$lib timeout 300 python bench.py --workload cfg3 --points asym2_q191_fft,full_fft --opt fft_n=$n --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02/fft_$(basename $lib .so)_$n.json 2>&1
  done
done
python tools/pcie_probe.py > gpurun_out/r02/pcie.log 2>&1
python tools/e2e_check.py pg > gpurun_out/r02/e2e_check_pg.log 2>&1
