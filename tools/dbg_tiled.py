"""Development check of the tiled kernel on one case: python tools/dbg_tiled.py L N W_block packing Q [T]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle as O
from paper_1201_3018_b200 import binding as pcb

L, N, Wb, pk, Q = (int(x) for x in sys.argv[1:6])
T = int(sys.argv[6]) if len(sys.argv) > 6 else 0
rng = np.random.default_rng(1)
s = np.clip(rng.laplace(0, 0.2, L), -1, 1)
k = rng.uniform(-1, 1, N)
dev = torch.device("cuda")
opts = pcb.opts_default(rmax_rule=1, bound_policy=pcb.BOUND_WARN)
opts.reserved[1] = T
with pcb.Plan(L, N, Wb, 0, pk, Q, opts=opts) as p:
    p.set_kernel(torch.from_numpy(k).to(dev))
    S = torch.from_numpy(s).to(dev)
    R = torch.full((L + N - 1,), float("nan"), dtype=torch.float64, device=dev)
    for i in range(3):
        p.execute(S, R)
    torch.cuda.synchronize()
    t0 = time.time()
    for i in range(10):
        p.execute(S, R)
    torch.cuda.synchronize()
    dt = (time.time() - t0) / 10
    got = R.cpu().numpy()
    info = p.info()
if pk == 0:
    ref = O.full_precision(s, k)
    err = float(np.max(np.abs(got - ref)) / np.max(np.abs(ref)))
    ok = err < 1e-12
else:
    ref = O.conv_pipeline(s, k, Wb, [0, O.SYM, O.ASYM2, O.ASYM3][pk], Q, rmax_rule=O.RMAX_L1).out
    bad = np.flatnonzero(~(got == ref))
    err = len(bad)
    ok = err == 0
    if not ok:
        print("first bad", bad[:10], got[bad[:5]], ref[bad[:5]])
print(f"L={L} N={N} W={Wb} pk={pk} Q={Q} tile={info['core_tile']} ok={ok} err={err} {dt*1e6:.1f} us/exec")
