"""Gap between consecutive persistent launches: min CTA start of launch i+1 minus max CTA
end of launch i (globaltimer), vs the per-launch event time."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1201_3018_b200 import binding as pcb
from paper_1201_3018_b200 import workloads as WL
s, k = WL.cfg2(seed=0)
dev = torch.device("cuda")
S = torch.from_numpy(s).to(dev)
R = torch.empty(len(s) + len(k) - 1, dtype=torch.float64, device=dev)
cases = [("asym2", 2, 511, 1, c) for c in (2, 3, 4)] + [("sym", 1, 127, 1, 4)] + [("full", 0, 0, 0, c) for c in (1, 2)]
for name, pk, Q, rm, cap in cases:
    o = pcb.opts_default(rmax_rule=rm)
    o.reserved[2] = cap
    name = f"{name} cap{cap}"
    with pcb.Plan(len(s), len(k), 4096, 0, pk, Q, opts=o) as p:
        p.set_kernel(torch.from_numpy(k).to(dev))
        recs = [torch.zeros(4 * 148 * 32, dtype=torch.int64, device=dev) for _ in range(6)]
        for _ in range(3): p.execute(S, R)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        gs = [pcb.execute_profile(p.h, S, R, r) for r in recs]
        b.record(); torch.cuda.synchronize()
        spans = []
        for g, r in zip(gs, recs):
            x = r[:4 * g].view(g, 4).cpu().numpy()
            spans.append((x[:, 1].min(), x[:, 2].max()))
        lens = [(e - s_) / 1e3 for s_, e in spans]
        gaps = [(spans[i + 1][0] - spans[i][1]) / 1e3 for i in range(len(spans) - 1)]
        ends = [(r[:4 * g].view(g, 4).cpu().numpy()) for g, r in zip(gs, recs)]
        last = ends[-1]
        t0 = last[:, 1].min()
        print(name, "grid", gs[0], "event us/launch %.1f" % (a.elapsed_time(b) / len(recs) * 1e3),
              "last-launch CTA starts %.1f..%.1f ends %.1f..%.1f us" % ((last[:, 1].min() - t0) / 1e3, (last[:, 1].max() - t0) / 1e3,
                                                                  (last[:, 2].min() - t0) / 1e3, (last[:, 2].max() - t0) / 1e3))
