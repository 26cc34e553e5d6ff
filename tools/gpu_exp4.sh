#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bA.log 2>&1
timeout 200 python bench.py --no-cpu-baseline --points asym2_10b,sym_8b,full > gpurun_out/v_A.json 2>/dev/null
PC_NVCC_EXTRA="-DPC_CONS_WARPS=12" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bB.log 2>&1
timeout 200 python bench.py --no-cpu-baseline --points asym2_10b,sym_8b,full > gpurun_out/v_B.json 2>/dev/null
timeout 200 python bench.py --no-cpu-baseline --points asym2_10b,sym_8b,full --opt 1=16 > gpurun_out/v_B16.json 2>/dev/null
timeout 300 python -m pytest tests -m gpu -x -q -k "bit_exact_pow2 or every_core_tile or parts_per_job" > gpurun_out/v_B_pt.log 2>&1
