"""Per-CTA timeline of the tiled persistent kernel (conv_execute_profile): how many CTAs are
resident per SM over time, per-job core durations, fill, and consumer cycle split.
    python tools/tiled_timeline.py [workload=cfg2] [L] > out.json
    PC_OPT="core_variant=1,parts_per_job=4" sets named conv_opts fields (e.g. core_variant=1: the FP64 FMA core)"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1201_3018_b200 import binding as pcb
from paper_1201_3018_b200 import workloads as WL

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
L = int(sys.argv[2]) if len(sys.argv) > 2 else 0
if wl == "cfg2":
    s, k = WL.cfg2(seed=0, L=L or (1 << 22))
    W_block = 4096
    points = {"asym2_10b": (2, 511, 1), "sym_8b": (1, 127, 1), "full": (0, 0, 0)}
elif wl == "cfg3":
    s, k = WL.cfg3(seed=0, L=L or (1 << 22))
    W_block = 16384
    points = {"asym2_9b": (2, 255, 1), "full": (0, 0, 0)}
else:
    s, k = WL.cfg5(seed=0, L=L or (1 << 24))
    W_block = 4096
    points = {"asym2_q535": (2, 535, 1), "full": (0, 0, 0)}
dev = torch.device("cuda")
S, R = torch.from_numpy(s).to(dev), torch.empty(len(s) + len(k) - 1, dtype=torch.float64, device=dev)
NC = 148 * 32
KTW = 24 * NC
KTP = KTW + 148 * 16 * 16 * 4
rec = torch.zeros(KTP + 148 * 4 * 16 * 4, dtype=torch.int64, device=dev)
out = {}
for name, (pk, Q, rm) in points.items():
    o = pcb.opts_default(rmax_rule=rm)
    for kv in filter(None, os.environ.get("PC_OPT", "").split(",")):
        f, v = kv.split("=")
        setattr(o, f, int(v))
    with pcb.Plan(len(s), len(k), W_block, 0, pk, Q, opts=o) as p:
        p.set_kernel(torch.from_numpy(k).to(dev))
        for _ in range(3):
            p.execute(S, R)
        rec.zero_()
        g = pcb.execute_profile(p.h, S, R, rec)
        torch.cuda.synchronize()
        info = p.info()
        a = rec.cpu().numpy()
    r = a[:4 * g].reshape(g, 4)
    c = a[4 * NC:4 * NC + 4 * g].reshape(g, 4).astype(float)
    tr = a[8 * NC:8 * NC + 16 * g].reshape(g, 16)
    t0 = r[:, 1].min()
    st, en = (r[:, 1] - t0) / 1e3, (r[:, 2] - t0) / 1e3
    T_end = en.max()
    # resident CTAs per SM over time (0.5 us bins)
    bins = np.arange(0, T_end + 0.5, 0.5)
    occ = np.zeros((148, len(bins)))
    for smid, a_, b_ in zip(r[:, 0], st, en):
        occ[smid % 148, (bins >= a_) & (bins < b_)] += 1
    hist = {int(v): round(float(np.mean(occ == v)), 4) for v in np.unique(occ)}
    sm_end = np.array([en[r[:, 0] == sm].max() for sm in np.unique(r[:, 0])])
    jobdur = []
    for i in range(g):
        prev = r[i, 1] + c[i, 3]
        for j in range(min(16, int(r[i, 3]))):
            if tr[i, j]:
                jobdur.append((tr[i, j] - prev) / 1e3)
                prev = tr[i, j]
    W = a[KTW:KTP].reshape(148, 16, 16, 4)[:g]
    Pr = a[KTP:KTP + 148 * 4 * 16 * 4].reshape(148, 4, 16, 4)[:g]
    # per SMSP: how many warps are in their core phase over time (0.25 us bins); DMMA core: from
    # the core-token acquisition (wait recorded in the high word of the sequence) to core done
    tb = np.arange(0, T_end + 0.25, 0.25)
    act = np.zeros((g, 4, len(tb)))
    for cc in range(g):
        for w in range(16):
            for j in range(16):
                if W[cc, w, j, 1] == 0 or W[cc, w, j, 2] == 0:
                    continue
                a0, b0_ = (W[cc, w, j, 1] - t0) / 1e3, (W[cc, w, j, 2] - t0) / 1e3
                a0 += ((int(W[cc, w, j, 0]) >> 32) * 16) / 1e3
                act[cc, (w + 4) % 4, (tb >= a0) & (tb < b0_)] += 1
    cta_end = {cc: (r[cc, 2] - t0) / 1e3 for cc in range(g)}
    live = np.array([[tb < cta_end[cc]] * 4 for cc in range(g)]).reshape(g, 4, len(tb))
    hist_core = {int(v): round(float(np.sum((act == v) & live) / np.sum(live)), 4) for v in range(5)}
    # where the zero-warps-in-core SMSP time sits: before the first core, between cores, after the last
    zero = (act == 0) & live
    any_core = act > 0
    first = np.argmax(any_core, axis=2)
    last = act.shape[2] - 1 - np.argmax(any_core[:, :, ::-1], axis=2)
    idx = np.arange(act.shape[2])[None, None, :]
    zsplit = {"before_first_core": float(np.sum(zero & (idx < first[:, :, None]))),
              "between_cores": float(np.sum(zero & (idx >= first[:, :, None]) & (idx <= last[:, :, None]))),
              "after_last_core": float(np.sum(zero & (idx > last[:, :, None])))}
    ztot = max(1.0, float(np.sum(live)))
    zsplit = {k: round(v / ztot, 4) for k, v in zsplit.items()}
    def cta_trace(c):
        def prow(w, j):
            v = int(Pr[c, w, j, 0])
            tc = (Pr[c, w, j, 2] - t0) / 1e3
            tr_ = tc + ((v >> 16) & 0xffff) * 16 / 1e3          # raw block landed (raw-staged producers)
            tp = tr_ + ((v >> 32) & 0xffff) * 16 / 1e3
            return [v & 0xffff, w, round((Pr[c, w, j, 1] - t0) / 1e3, 1), round(tc, 1), round(tr_, 1), round(tp, 1),
                    round(tp + (v >> 48) * 16 / 1e3, 1), round((Pr[c, w, j, 3] - t0) / 1e3, 1)]
        diag = Pr[c, 1, :, 0] > (1 << 50)            # raw-staged producers: warp 1's slots hold peak-phase stamps
        prod = [prow(w, j) for w in range(4) for j in range(15)
                if Pr[c, w, j, 3] and not (w == 1 and diag[j]) and not (int(Pr[c, w, j, 0]) >> 62) & 1]
        pdiag = [[j] + [round((Pr[c, 1, j, i] - t0) / 1e3, 2) for i in range(4)] for j in range(15) if diag[j]]
        cons = [[w, int(W[c, w, j, 0]) & 0xffffffff, round((W[c, w, j, 1] - t0) / 1e3, 1),
                 round((W[c, w, j, 1] - t0) / 1e3 + ((int(W[c, w, j, 0]) >> 32) * 16) / 1e3, 1),
                 round((W[c, w, j, 2] - t0) / 1e3, 1), round((W[c, w, j, 3] - t0) / 1e3, 1)]
                for w in range(16) for j in range(16) if W[c, w, j, 1]]
        return {"produced[mseq,warp,t_start,t_claimed,t_raw,t_peak,t_slot,t_pub]": sorted(prod),
                "peak_diag[j,t_local_max,t_reduced,t_cs,t_inv]": pdiag,
                "consumed[warp,mseq,t_ready,t_in_core,t_core_done,t_stored]": sorted(cons, key=lambda x: x[2])}
    fill_phases = (Pr[:, :, 15, :3].astype(float) - r[:, 1][:, None, None]) / 1e3   # claimed, peak, packed (us)
    fill_stats = {k: round(float(np.median(fill_phases[:, :, i])), 2) for i, k in enumerate(["claimed", "peak", "packed"])}
    # producer CTAs (producer-SM mode): records with bit 62 set in producer-record slot 0
    pm = (Pr[:, :, :, 0].astype(np.uint64) >> np.uint64(62)) & np.uint64(1)
    prod_cta = None
    if pm.any():
        sel = pm.astype(bool)
        tcl, traw, tdone = Pr[:, :, :, 1][sel], Pr[:, :, :, 2][sel], Pr[:, :, :, 3][sel]
        prod_cta = {"jobs_recorded": int(sel.sum()), "ctas": int(np.any(sel.reshape(g, -1), axis=1).sum()),
                    "claim_to_raw_us_median": round(float(np.median((traw - tcl) / 1e3)), 2),
                    "raw_to_flag_us_median": round(float(np.median((tdone - traw) / 1e3)), 2),
                    "first_flag_us": round(float((tdone.min() - t0) / 1e3), 2),
                    "last_flag_us": round(float((tdone.max() - t0) / 1e3), 2)}
    crit = int(np.argmax(r[:, 2]))                  # the CTA that ends last
    out[name] = {"producer_ctas": prod_cta, "cta_last": crit, "cta_last_trace": cta_trace(crit), "zero_core_time_split": zsplit, "fill_phases_us_median": fill_stats, "smsp_warps_in_core_time_frac": hist_core, "cta0": cta_trace(0), "grid": g, "tile": info["core_tile"], "kernel_us": float(T_end),
                 "start_spread_us": float(st.max()), "sm_end_min_us": float(sm_end.min()),
                 "sm_end_median_us": float(np.median(sm_end)), "sm_end_max_us": float(sm_end.max()),
                 "resident_ctas_per_sm_time_frac": hist,
                 "jobs_per_cta_hist": np.bincount(r[:, 3]).tolist(),
                 "fill_us_mean": float(c[:, 3].mean() / 1e3),
                 "job_core_us": {"min": float(np.min(jobdur)), "median": float(np.median(jobdur)),
                                 "max": float(np.max(jobdur))} if jobdur else None,
                 "consumer_w0_cycles_frac": dict(zip(["wait_full", "core", "unpack_store"],
                                                     np.round(c[:, :3].sum(0) / max(1.0, c[:, :3].sum()), 3).tolist())),
                 "trace_cta0_us": [round((x - t0) / 1e3, 2) for x in tr[0] if x],
                 "trace_cta_last_us": [round((x - t0) / 1e3, 2) for x in tr[g - 1] if x]}
print(json.dumps(out, indent=1))
