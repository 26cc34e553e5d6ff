"""Per-CTA timeline of the persistent kernel (conv_execute_profile): when each SM's CTAs
start/finish and how many blocks they processed -> quantifies fill/tail/imbalance."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1201_3018_b200 import binding as pcb
from paper_1201_3018_b200 import workloads as WL

points = {"asym2_10b": (2, 511, 1), "sym_8b": (1, 127, 1), "full": (0, 0, 0)}
L = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 22)
s, k = WL.cfg2(seed=0, L=L)
dev = torch.device("cuda")
S, R = torch.from_numpy(s).to(dev), torch.empty(len(s) + len(k) - 1, dtype=torch.float64, device=dev)
rec = torch.zeros(24 * 148 * 32, dtype=torch.int64, device=dev)
out = {}
for name, (pk, Q, rm) in points.items():
    with pcb.Plan(len(s), len(k), 4096, 0, pk, Q, rmax_rule=rm) as p:
        p.set_kernel(torch.from_numpy(k).to(dev))
        for _ in range(3):
            p.execute(S, R)
        g = pcb.execute_profile(p.h, S, R, rec)
        torch.cuda.synchronize()
        r = rec[:4 * g].view(g, 4).cpu().numpy()
        c = rec[4 * 148 * 32:4 * 148 * 32 + 4 * g].view(g, 4).cpu().numpy().astype(float)
        tr = rec[8 * 148 * 32:8 * 148 * 32 + 16 * g].view(g, 16).cpu().numpy()
    t0 = r[:, 1].min()
    st, en = (r[:, 1] - t0) / 1e3, (r[:, 2] - t0) / 1e3
    sm_end = {}
    for smid, e_ in zip(r[:, 0], en):
        sm_end[smid] = max(sm_end.get(smid, 0), e_)
    ends = np.array(list(sm_end.values()))
    out[name] = {"grid": g, "kernel_us": float(en.max()), "start_spread_us": float(st.max()),
                 "sm_end_min_us": float(ends.min()), "sm_end_median_us": float(np.median(ends)),
                 "idle_frac": float(1 - ends.mean() / en.max()),
                 "blocks_per_cta": np.bincount(r[:, 3]).tolist(),
                 "consumer_cycles_frac": dict(zip(["wait_full", "core", "decode_store"],
                                                  np.round(c[:, :3].sum(0) / c[:, :3].sum(), 3).tolist())),
                 "fill_us_mean": float(c[:, 3].mean() / 1e3),
                 "fill_peak_us_mean": float(c[:, 2].mean() / 1e3),
                 "consumer_cycles_mean": np.round(c.mean(0)).tolist(),
                 "trace_cta0_us": [round((x - r[0, 1]) / 1e3, 2) if x else None for x in tr[0]],
                 "trace_cta300_us": [round((x - r[min(300, g - 1), 1]) / 1e3, 2) if x else None for x in tr[min(300, g - 1)]],
                 "cta0_end_us": round((r[0, 2] - r[0, 1]) / 1e3, 2)}
print(json.dumps(out, indent=1))
