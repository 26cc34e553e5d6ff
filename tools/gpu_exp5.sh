#!/bin/bash
mkdir -p gpurun_out
PC_NVCC_EXTRA="-DPC_CONS_WARPS=8" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bC.log 2>&1
timeout 200 python bench.py --no-cpu-baseline --points asym2_10b,sym_8b,full > gpurun_out/v_C.json 2>/dev/null
timeout 200 python bench.py --no-cpu-baseline --points asym2_10b,sym_8b,full --opt 1=16 > gpurun_out/v_C16.json 2>/dev/null
PC_NVCC_EXTRA="-DPC_CONS_WARPS=12 -DPC_PROD_WARPS=2" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bD.log 2>&1
timeout 200 python bench.py --no-cpu-baseline --points asym2_10b,sym_8b,full > gpurun_out/v_D.json 2>/dev/null
PC_NVCC_EXTRA="-DPC_CONS_WARPS=12" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bB.log 2>&1
timeout 300 python tools/tiled_timeline.py cfg2 > gpurun_out/tl_B.json 2>/dev/null
