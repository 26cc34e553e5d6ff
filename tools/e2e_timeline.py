"""Replica of conv_execute_host's pipeline (H2D / compute / D2H of block ranges on three
streams) with timing events, to see where an e2e step's time goes (cfg2 asym2 10-bit)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1201_3018_b200 import binding as pcb
from paper_1201_3018_b200 import workloads as WL

s, k = WL.cfg2(seed=0)
L, N = len(s), len(k)
dev = torch.device("cuda")
sh = torch.from_numpy(s).pin_memory()
rh = torch.empty(L + N - 1, dtype=torch.float64).pin_memory()
d_in = torch.empty(L, dtype=torch.float64, device=dev)
d_out = torch.empty(L + N - 1, dtype=torch.float64, device=dev)
sc, s1, s2 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
W = [1, 2, 4, 4, 4, 4, 4, 2, 1]
cum = np.concatenate([[0], np.cumsum(W)])
with pcb.Plan(L, N, 4096, 0, 2, 511, rmax_rule=1) as p:
    p.set_kernel(torch.from_numpy(k).to(dev))
    info = p.info()
    P, Wo, Np, Wb = info["P"], info["W"], info["Np"], info["W_block"]

    def run(ev):
        in_done, out_done = 0, 0
        start = torch.cuda.Event(enable_timing=True)
        start.record(sc)
        s1.wait_stream(sc)
        s2.wait_stream(sc)
        for c in range(9):
            b0, b1 = P * cum[c] // cum[9], P * cum[c + 1] // cum[9]
            last = b1 - 1
            in_end = min(L, (0 if last == 0 else last * Wo - 2) + Wb) if c < 8 else L
            out_end = min(L + N - 1, (L + N - 1) if b1 == P else Np - 1 + b1 * Wo)
            e = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
            with torch.cuda.stream(s1):
                e[0].record(s1)
                d_in[in_done:in_end].copy_(sh[in_done:in_end], non_blocking=True)
                e[1].record(s1)
            in_done = in_end
            sc.wait_event(e[1])
            with torch.cuda.stream(sc):
                e[2].record(sc)
                pcb.execute_blocks(p.h, d_in, 0, d_out, 0, int(b0), int(b1))
                e[3].record(sc)
            s2.wait_event(e[3])
            with torch.cuda.stream(s2):
                e[4].record(s2)
                rh[out_done:out_end].copy_(d_out[out_done:out_end], non_blocking=True)
                e[5].record(s2)
            out_done = out_end
            ev.append(e)
        sc.wait_stream(s2)
        end = torch.cuda.Event(enable_timing=True)
        end.record(sc)
        return start, end

    for _ in range(3):
        run([])
    torch.cuda.synchronize()
    ev = []
    st, en = run(ev)
    torch.cuda.synchronize()
    print(f"total {st.elapsed_time(en):.3f} ms")
    for c, e in enumerate(ev):
        t = [st.elapsed_time(x) for x in e]
        print(f"chunk {c}: h2d {t[0]:.3f}-{t[1]:.3f}  core {t[2]:.3f}-{t[3]:.3f}  d2h {t[4]:.3f}-{t[5]:.3f}")
