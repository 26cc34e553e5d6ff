"""Zero-copy variants of the cfg2 asym2 host-buffer step (diagnostics): the conv kernels reading
the pinned host input and/or writing the pinned host output directly (UVA pointers), with and
without the prepack kernel, against the copy pipeline (conv_execute_host_blocks).
    python tools/zero_copy_probe.py"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1201_3018_b200 import binding as pcb
from paper_1201_3018_b200 import workloads as WL

s, k = WL.cfg2(seed=0)
dev = torch.device("cuda")
out = {}
lib = pcb.load()
sh = torch.from_numpy(s).pin_memory()
ref = None
for prepack in (0, 1):
    o = pcb.opts_default(rmax_rule=1, prepack=prepack)
    with pcb.Plan(len(s), len(k), 4096, 0, 2, 511, opts=o) as p:
        p.set_kernel(torch.from_numpy(k).to(dev))
        info = p.info()
        L_out, P = info["L_out"], info["P"]
        rh = torch.empty(L_out, dtype=torch.float64).pin_memory()
        d_in = torch.from_numpy(s).to(dev)
        d_out = torch.empty(L_out, dtype=torch.float64, device=dev)
        st = torch.cuda.current_stream().cuda_stream

        def timeit(fn, reps=10):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(reps):
                fn()
            torch.cuda.synchronize()
            return (time.perf_counter() - t0) * 1e3 / reps

        variants = {
            "device_only": lambda: lib.conv_execute(p.h, d_in.data_ptr(), d_out.data_ptr(), st),
            "zc_in": lambda: lib.conv_execute(p.h, sh.data_ptr(), d_out.data_ptr(), st),
            "zc_out": lambda: lib.conv_execute(p.h, d_in.data_ptr(), rh.data_ptr(), st),
            "zc_both": lambda: lib.conv_execute(p.h, sh.data_ptr(), rh.data_ptr(), st),
            "copy_pipeline": lambda: lib.conv_execute_host_blocks(p.h, sh.data_ptr(), 0, rh.data_ptr(), 0, 0, P, st),
        }
        # hybrid: the pack kernels read the pinned input in place (zero-copy), the copy engine
        # brings each block range's outputs back while the next range computes
        s_cmp, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()
        W, Np = info["W"], info["Np"]

        def out_end(b1):
            return L_out if b1 == P else min(Np - 1 + b1 * W, L_out)

        def hybrid(wts):
            cum = [0]
            for w_ in wts:
                cum.append(cum[-1] + w_)
            cur = torch.cuda.current_stream()
            s_cmp.wait_stream(cur)
            s_d2h.wait_stream(cur)
            o_done = 0
            for c in range(len(wts)):
                b0, b1 = P * cum[c] // cum[-1], P * cum[c + 1] // cum[-1]
                lib.conv_execute_blocks(p.h, sh.data_ptr(), 0, d_out.data_ptr(), 0, b0, b1, s_cmp.cuda_stream)
                ev = torch.cuda.Event()
                ev.record(s_cmp)
                s_d2h.wait_event(ev)
                oe = out_end(b1)
                with torch.cuda.stream(s_d2h):
                    rh[o_done:oe].copy_(d_out[o_done:oe], non_blocking=True)
                o_done = oe
            cur.wait_stream(s_cmp)
            cur.wait_stream(s_d2h)

        for wname, wts in (("h1", [1]), ("h4", [1] * 4), ("h8", [1] * 8), ("h16", [1] * 16),
                           ("hr8", [1, 2, 3, 3, 3, 3, 2, 1]), ("hl15", [1, 1] + [2] * 11 + [1, 1])):
            gs = torch.cuda.Stream()
            with torch.cuda.stream(gs):
                hybrid(wts)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=gs):
                hybrid(wts)
            variants[f"hybrid_{wname}"] = g.replay
        for name, fn in variants.items():
            ms = timeit(fn)
            torch.cuda.synchronize()
            rh_ = rh.numpy().copy()
            got = (d_out.cpu().numpy() if name in ("device_only", "zc_in") else rh_)
            rh.fill_(float("nan"))
            if ref is None:
                ref = got.copy()
            out[f"prepack{prepack}_{name}_ms"] = round(ms, 4)
            out[f"prepack{prepack}_{name}_same"] = bool(np.array_equal(got, ref))
print(json.dumps(out, indent=1))
