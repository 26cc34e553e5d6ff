"""conv_execute_host timing (cfg2 asym2 10-bit): mean per call over 20 calls, host wall and
CUDA events, for the chunking in effect (PC_HOST_CHUNKS)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1201_3018_b200 import binding as pcb
from paper_1201_3018_b200 import workloads as WL

s, k = WL.cfg2(seed=0)
dev = torch.device("cuda")
sh = torch.from_numpy(s).pin_memory()
rh = torch.empty(len(s) + len(k) - 1, dtype=torch.float64).pin_memory()
with pcb.Plan(len(s), len(k), 4096, 0, 2, 511, rmax_rule=1) as p:
    p.set_kernel(torch.from_numpy(k).to(dev))
    for _ in range(3):
        p.execute_host(sh, rh)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record()
    for _ in range(20):
        p.execute_host(sh, rh)
    e1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / 20
print(f"chunks={os.environ.get('PC_HOST_CHUNKS', 'default')} events {e0.elapsed_time(e1) / 20:.3f} ms  wall {wall * 1e3:.3f} ms")
