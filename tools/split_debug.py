"""Producer-SM mode smoke: one cfg2-geometry launch, compared with the fused path (bit-exact)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1201_3018_b200 import binding as pcb
from paper_1201_3018_b200 import workloads as WL
L = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 20)
P = int(sys.argv[2]) if len(sys.argv) > 2 else 4
s, k = WL.cfg2(seed=0, L=L)
dev = torch.device("cuda")
S = torch.from_numpy(s).to(dev)
outs = {}
for name, pre in (("fused", 0), ("split", -P)):
    o = pcb.opts_default(rmax_rule=1)
    o.prepack = pre
    with pcb.Plan(L, len(k), 4096, 0, 2, 511, opts=o) as p:
        p.set_kernel(torch.from_numpy(k).to(dev))
        R = torch.full((L + len(k) - 1,), float("nan"), dtype=torch.float64, device=dev)
        for _ in range(3):
            try:
                p.execute(S, R)
                torch.cuda.synchronize()
            except Exception as ex:
                print(name, "error", ex)
                break
        outs[name] = R.cpu().numpy()
a, b = outs["fused"], outs["split"]
print("equal", np.array_equal(a, b), "nan", int(np.isnan(b).sum()), "diff", int(np.sum(a != b)))
