"""Repro: early_fill = 1 through conv_execute_host_blocks (chunked launches back to back)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1201_3018_b200 import binding as pcb
from paper_1201_3018_b200 import workloads as WL
pk = int(sys.argv[1]) if len(sys.argv) > 1 else 2
Q = int(sys.argv[2]) if len(sys.argv) > 2 else 511
raw = int(sys.argv[3]) if len(sys.argv) > 3 else 0
s, k = WL.cfg2(seed=0)
o = pcb.opts_default(rmax_rule=1, early_fill=1, raw_staging=raw)
with pcb.Plan(len(s), len(k), 4096, 0, pk, Q, opts=o) as p:
    p.set_kernel(torch.from_numpy(k).cuda())
    sh = torch.from_numpy(s).pin_memory()
    rh = torch.empty(p.info()["L_out"], dtype=torch.float64).pin_memory()
    for i in range(5):
        p.execute_host_blocks(sh, 0, rh, 0, 0, p.info()["P"])
        print("ok", i, flush=True)
