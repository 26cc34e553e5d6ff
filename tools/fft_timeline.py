"""Per-job phase times of the FFT core (conv_execute_profile on an FFT plan): median us of
peak, packing, forward FFT, spectrum product, inverse FFT, unpack+store.
    python tools/fft_timeline.py [L] [fft_n ...]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1201_3018_b200 import binding as pcb
from paper_1201_3018_b200 import workloads as WL

L = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 22)
s, k = WL.cfg3(seed=0, L=L)
dev = torch.device("cuda")
S, R = torch.from_numpy(s).to(dev), torch.empty(len(s) + len(k) - 1, dtype=torch.float64, device=dev)
rec = torch.zeros(8 * 4096 + 64, dtype=torch.int64, device=dev)
out = {}
sizes = [int(x) for x in sys.argv[2:]] or [0]
cases = {f"{nm}_n{n}": (pk, Q, rm, n) for n in sizes for nm, (pk, Q, rm) in
         {"asym2_q191": (2, 191, 1), "full": (0, 0, 0)}.items()}
for name, (pk, Q, rm, fn) in cases.items():
    opts = pcb.opts_default(rmax_rule=rm, core=1, fft_n=fn)
    with pcb.Plan(len(s), len(k), 16384, 0, pk, Q, opts=opts) as p:
        p.set_kernel(torch.from_numpy(k).to(dev))
        for _ in range(3):
            p.execute(S, R)
        rec.zero_()
        g = pcb.execute_profile(p.h, S, R, rec)
        torch.cuda.synchronize()
        n = min(g, 4096)
        a = rec[:8 * n].view(n, 8).cpu().numpy().astype(np.int64)
        a = a[a[:, 7] != 0]                                  # records of jobs that exist
        fft_n = p.info()["fft_n"]
    d = np.diff(a[:, 1:], axis=1) / 1e3
    t0 = a[:, 1].min()
    out[name] = {"fft_n": fft_n, "jobs": int(g), "kernel_us": float((a[:, 7].max() - t0) / 1e3),
                 "phase_us_median": dict(zip(["peak", "pack", "fwd_fft", "product", "inv_fft", "unpack_store"],
                                             np.round(np.median(d, axis=0), 2).tolist())),
                 "job_us_median": float(np.median((a[:, 7] - a[:, 1]) / 1e3))}
print(json.dumps(out, indent=1))
