"""Host cost of one conv_execute call (binding + C ABI + launch) on a small plan whose GPU time
is far below it: time N back-to-back calls with a host clock and with CUDA events."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1201_3018_b200 import binding as pcb

dev = torch.device("cuda")
for L, W, packing, Q in ((1 << 16, 4096, 2, 511), (1 << 22, 4096, 2, 511)):
    s = torch.randn(L, dtype=torch.float64, device=dev).clamp_(-1, 1)
    k = torch.randn(513, dtype=torch.float64, device=dev) / 20
    r = torch.empty(L + 512, dtype=torch.float64, device=dev)
    with pcb.Plan(L, 513, W, 0, packing, Q, rmax_rule=1) as p:
        p.set_kernel(k)
        for _ in range(10):
            p.execute(s, r)
        torch.cuda.synchronize()
        n = 200
        t0 = time.perf_counter()
        for _ in range(n):
            p.execute(s, r)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        st = torch.cuda.current_stream().cuda_stream
        t3 = time.perf_counter()
        for _ in range(n):
            pcb.execute(p.h, s, r, st)
        t4 = time.perf_counter()
        torch.cuda.synchronize()
        t5 = time.perf_counter()
        print(f"L={L}: submit {1e6 * (t1 - t0) / n:.1f} us/call (Plan.execute), {1e6 * (t4 - t3) / n:.1f} us/call "
              f"(explicit stream); total {1e6 * (t2 - t0) / n:.1f} / {1e6 * (t5 - t3) / n:.1f} us/call incl. GPU")
