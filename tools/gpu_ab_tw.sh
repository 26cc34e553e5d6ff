P=gpurun_out/r02d_pkx; mkdir -p $P
timeout 600 python -m pytest tests -m gpu -q -k "fft or backend" > $P/pytest_fft.log 2>&1; echo "rc=$?" >> $P/pytest_fft.log
bash tools/gpu_ab_fft.sh r02d_pkx "base pkx" 3
