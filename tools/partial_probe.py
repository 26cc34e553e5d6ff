import sys, torch, numpy as np
sys.path.insert(0, ".")
from paper_1201_3018_b200 import binding as pcb
from paper_1201_3018_b200 import workloads as WL
s, k = WL.cfg2(seed=0)
L, N = len(s), len(k)
dev = torch.device("cuda")
S = torch.from_numpy(s).to(dev); R = torch.empty(L + N - 1, dtype=torch.float64, device=dev)
with pcb.Plan(L, N, 4096, 0, 2, 511, rmax_rule=1) as p:
    p.set_kernel(torch.from_numpy(k).to(dev))
    P = p.info()["P"]
    for nb in (48, 98, 195, 585, 1171):
        for _ in range(3): pcb.execute_blocks(p.h, S, 0, R, 0, 0, nb)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): pcb.execute_blocks(p.h, S, 0, R, 0, 0, nb)
        e1.record(); torch.cuda.synchronize()
        e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2.record()
        for _ in range(20): pcb.execute_blocks(p.h, S, 0, R, 0, 500, 500 + min(nb, 671))
        e3.record(); torch.cuda.synchronize()
        print(nb, "from 0: %.1f us" % (e0.elapsed_time(e1) / 20 * 1e3), " from 500: %.1f us" % (e2.elapsed_time(e3) / 20 * 1e3))
