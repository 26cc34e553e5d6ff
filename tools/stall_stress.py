"""Stress (mode 2: conv_execute_host_blocks calls): many back-to-back persistent launches (cfg2 geometry) on one stream, no host sync in
between, alternating input/output buffers; reports any watchdog status (diagnostics).
    python tools/stall_stress.py [packing=2] [Q=511] [early_fill=1] [raw_staging=0] [n=2000] [graph=0]"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1201_3018_b200 import binding as pcb
from paper_1201_3018_b200 import workloads as WL

a = [int(x) for x in sys.argv[1:]] + [None] * 6
pk, Q, ef, raw, n, graph = [v if v is not None else d for v, d in zip(a[:6], (2, 511, 1, 0, 2000, 0))]
s, k = WL.cfg2(seed=0)
o = pcb.opts_default(rmax_rule=1, early_fill=ef, raw_staging=raw)
with pcb.Plan(len(s), len(k), 4096, 0, pk, Q, opts=o) as p:
    p.set_kernel(torch.from_numpy(k).cuda())
    L_out = p.info()["L_out"]
    S = [torch.from_numpy(s).cuda(), torch.from_numpy(s[::-1].copy()).cuda()]
    R = [torch.empty(L_out, dtype=torch.float64, device="cuda") for _ in range(2)]
    t0 = time.time()
    bad = 0
    sh = torch.from_numpy(s).pin_memory()
    rh = torch.empty(L_out, dtype=torch.float64).pin_memory()
    P = p.info()["P"]
    for i in range(n):
        try:
            if graph == 2:                               # host-buffer pipeline (chunked launches)
                p.execute_host_blocks(sh, 0, rh, 0, 0, P)
            else:
                p.execute(S[i & 1], R[i & 1])
        except pcb.PcError as ex:
            print("error at", i, ex, flush=True)
            bad += 1
            if bad > 3:
                break
        if i % 200 == 199:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    try:
        p.execute(S[0], R[0])
        torch.cuda.synchronize()
        p.execute(S[0], R[0])
    except pcb.PcError as ex:
        print("error at end", ex)
        bad += 1
    print(f"pk={pk} Q={Q} ef={ef} raw={raw} n={n} errors={bad} {time.time() - t0:.1f}s", flush=True)
