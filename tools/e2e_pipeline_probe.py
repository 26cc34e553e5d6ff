"""Where the host-buffer pipeline (conv_execute_host_blocks) loses time against the PCIe duplex
floor: the same three-stream pipeline rebuilt in Python around conv_execute_blocks, with timing
events on every stage, and variants (copies only / device copy instead of the conv kernel /
the conv kernel).  Prints per-variant ms per step and one chunk timeline (diagnostics).
    python tools/e2e_pipeline_probe.py"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1201_3018_b200 import binding as pcb
from paper_1201_3018_b200 import workloads as WL

s, k = WL.cfg2(seed=0)
dev = torch.device("cuda")
L = len(s)
out = {}
with pcb.Plan(L, len(k), 4096, 0, 2, 511, rmax_rule=1) as p:
    p.set_kernel(torch.from_numpy(k).to(dev))
    info = p.info()
    P, L_out, W, Np = info["P"], info["L_out"], info["W"], info["Np"]
    sh = torch.from_numpy(s).pin_memory()
    rh = torch.empty(L_out, dtype=torch.float64).pin_memory()
    d_in = torch.empty(L, dtype=torch.float64, device=dev)
    d_out = torch.empty(L_out, dtype=torch.float64, device=dev)
    d_tmp = torch.zeros(L_out, dtype=torch.float64, device=dev)
    s_h2d, s_cmp, s_d2h = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()

    def in_end(b1):
        last = b1 - 1
        return min((0 if last == 0 else last * W - 2) + 4096, L)

    def out_end(b1):
        return L_out if b1 == P else min(Np - 1 + b1 * W, L_out)

    def run(weights, mode, rec=None):
        cum = [0]
        for w in weights:
            cum.append(cum[-1] + w)
        i_done = o_done = 0
        evs = []
        cur = torch.cuda.current_stream()
        s_h2d.wait_stream(cur)
        s_d2h.wait_stream(cur)
        s_cmp.wait_stream(cur)
        for c in range(len(weights)):
            b0, b1 = P * cum[c] // cum[-1], P * cum[c + 1] // cum[-1]
            ie, oe = in_end(b1), out_end(b1)
            t = [torch.cuda.Event(enable_timing=True) for _ in range(6)] if rec is not None else None
            with torch.cuda.stream(s_h2d):
                if t: t[0].record()
                if ie > i_done and mode != "nocopy":
                    d_in[i_done:ie].copy_(sh[i_done:ie], non_blocking=True)
                i_done = max(i_done, ie)
                e_in = torch.cuda.Event()
                e_in.record()
                if t: t[1].record()
            with torch.cuda.stream(s_cmp):
                s_cmp.wait_event(e_in)
                if t: t[2].record()
                if mode in ("conv", "nocopy"):
                    p.execute_blocks(d_in, 0, d_out, 0, b0, b1, stream=s_cmp)
                elif mode == "devcopy":
                    d_out[o_done:oe].copy_(d_tmp[o_done:oe])
                e_c = torch.cuda.Event()
                e_c.record()
                if t: t[3].record()
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(e_c)
                if t: t[4].record()
                if oe > o_done and mode != "nocopy":
                    rh[o_done:oe].copy_(d_out[o_done:oe], non_blocking=True)
                o_done = max(o_done, oe)
                if t: t[5].record()
            if t: evs.append(t)
        cur.wait_stream(s_h2d)
        cur.wait_stream(s_cmp)
        cur.wait_stream(s_d2h)
        if rec is not None:
            rec.extend(evs)

    def timeit(fn, reps=20):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    lib_w = [1, 1] + [2] * 11 + [1, 1]
    for name, wts in (("lib15", lib_w), ("eq8", [1] * 8), ("eq4", [1] * 4), ("eq16", [1] * 16), ("one", [1])):
        for mode in ("copies", "devcopy", "conv", "nocopy"):
            out[f"{name}_{mode}"] = round(timeit(lambda: run(wts, mode)), 4)
    out["lib_execute_host_blocks"] = round(timeit(lambda: p.execute_host_blocks(sh, 0, rh, 0, 0, P)), 4)
    # the same pipelines captured once in a CUDA graph (no Python enqueue cost between chunks)
    for name, wts in (("lib15", lib_w), ("eq8", [1] * 8), ("eq4", [1] * 4), ("eq2", [1] * 2), ("one", [1]),
                      ("ramp8", [1, 2, 3, 3, 3, 3, 2, 1])):
        for mode in ("copies", "conv", "nocopy"):
            gs = torch.cuda.Stream()
            with torch.cuda.stream(gs):
                run(wts, mode)                       # warm (allocations, plan state) outside capture
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=gs):
                run(wts, mode)
            out[f"graph_{name}_{mode}"] = round(timeit(lambda: g.replay()), 4)
    # host cost of enqueueing conv_execute_blocks through the raw C ABI (no Python checks)
    import time
    lib = pcb.load()
    cum = [0]
    for w_ in lib_w:
        cum.append(cum[-1] + w_)
    rngs = [(P * cum[c] // cum[-1], P * cum[c + 1] // cum[-1]) for c in range(len(lib_w))]
    hs = s_cmp.cuda_stream
    for rep in range(3):
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(s_cmp)
        h0 = time.perf_counter()
        for b0, b1 in rngs:
            lib.conv_execute_blocks(p.h, d_in.data_ptr(), 0, d_out.data_ptr(), 0, b0, b1, hs)
        h1 = time.perf_counter()
        g1.record(s_cmp)
        torch.cuda.synchronize()
        out[f"raw_blocks15_host_us_per_call_rep{rep}"] = round((h1 - h0) * 1e6 / len(rngs), 1)
        out[f"raw_blocks15_gpu_ms_rep{rep}"] = round(g0.elapsed_time(g1), 4)
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    for _ in range(20):
        lib.conv_execute(p.h, d_in.data_ptr(), d_out.data_ptr(), hs)
    h1 = time.perf_counter()
    torch.cuda.synchronize()
    out["raw_execute_host_us_per_call"] = round((h1 - h0) * 1e6 / 20, 1)
    h0 = time.perf_counter()
    for _ in range(5):
        lib.conv_execute_host_blocks(p.h, sh.data_ptr(), 0, rh.data_ptr(), 0, 0, P, hs)
    h1 = time.perf_counter()
    out["raw_host_blocks_wall_ms"] = round((h1 - h0) * 1e3 / 5, 4)
    # one timeline of the library-weight pipeline with the conv kernel
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record()
    rec = []
    run(lib_w, "conv", rec)
    torch.cuda.synchronize()
    out["timeline_us[h2d_start,h2d_end,cmp_start,cmp_end,d2h_start,d2h_end]"] = [
        [round(t0.elapsed_time(e) * 1e3, 1) for e in t] for t in rec]
print(json.dumps(out, indent=1))
