"""Backend-validation residuals of the FFT core (conv_plan_set_kernel) across
regimes at the cfg3 geometry (WARN policy: never refused), for choosing test cases.
    python tools/fft_validate_probe.py > out.json"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1201_3018_b200 import binding as pcb
from paper_1201_3018_b200 import workloads as WL

s, k = WL.cfg3(seed=0, L=1 << 18)
dev = torch.device("cuda")
kd = torch.from_numpy(k).to(dev)
out = []
for packing, Qs in ((2, (63, 127, 191, 255, 285)), (3, (5, 8, 12)), (1, (5, 8, 12))):
    for Q in Qs:
        for fn in (0, 8192):
            o = pcb.opts_default(core=pcb.CORE_FFT, rmax_rule=pcb.RMAX_L1, bound_policy=pcb.BOUND_WARN, fft_n=fn)
            try:
                with pcb.Plan(len(s), len(k), 16384, 0, packing, Q, opts=o) as p:
                    p.set_kernel(kd)
                    i = p.info()
                    r = torch.empty(i["L_out"], dtype=torch.float64, device=dev)
                    p.execute(torch.from_numpy(s).to(dev), r)
                    torch.cuda.synchronize()
                    res, rc = p.residual()
                    rec = dict(packing=packing, Q=Q, fft_n=i["fft_n"], R=i["R_max"], bound_ok=i["bound_ok"],
                               backend_resid=i["backend_resid"], backend_ok=i["backend_ok"], u_sys=i["u_sys_cal"],
                               data_resid=res)
            except Exception as ex:                     # noqa: BLE001
                rec = dict(packing=packing, Q=Q, fft_n=fn, error=str(ex))
            print(json.dumps(rec), flush=True)
            out.append(rec)
