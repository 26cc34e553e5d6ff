mkdir -p gpurun_out/r02
python tools/tiled_timeline.py cfg2 > gpurun_out/r02/tl_fill16.json 2> gpurun_out/r02/tl_fill16.err
PC_LIB_PATH=tools/variants/libpc_fill4.so python tools/tiled_timeline.py cfg2 > gpurun_out/r02/tl_fill4.json 2> gpurun_out/r02/tl_fill4.err
