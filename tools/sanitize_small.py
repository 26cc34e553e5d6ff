"""Small runs of every tiled-kernel variant for compute-sanitizer (memcheck / racecheck):
DMMA and FMA cores, all packings, conv and xcorr, tap chunks, parts per job 1/2/4."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1201_3018_b200 import binding as pcb

dev = torch.device("cuda")
rng = np.random.default_rng(0)
cases = [(20000, 513, 4096, 31), (9000, 100, 512, 15), (40000, 4096, 16384, 3)]
n = 0
for L, N, W, Q in cases:
    s = torch.from_numpy(np.clip(rng.laplace(0, 0.3, L), -1, 1)).to(dev)
    k = torch.from_numpy(rng.uniform(-1, 1, N)).to(dev)
    for packing in (0, 1, 2, 3):
        for core in (2, 1):
            for mode in (0, 1):
                for npart in ((0, 2) if N < 1000 else (0,)):
                    o = pcb.opts_default(bound_policy=1, exec=2, rmax_rule=1)
                    o.reserved[2], o.reserved[3] = core, npart
                    with pcb.Plan(L, N, W, mode, packing, 0 if packing == 0 else Q, opts=o) as p:
                        p.set_kernel(k)
                        r = torch.empty(p.info()["L_out"], dtype=torch.float64, device=dev)
                        p.execute(s, r)
                        torch.cuda.synchronize()
                        n += 1
print("runs", n, "ok")
