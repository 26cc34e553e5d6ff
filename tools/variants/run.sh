for h in 0 200 1000 20000; do echo "hint $h" >> gpurun_out/gap_var.log; PC_LIB_PATH=tools/variants/lib_h$h.so python tools/launch_gap.py >> gpurun_out/gap_var.log 2>&1; done
