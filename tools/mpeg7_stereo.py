"""the MPEG-7 stereo-descriptor regime of §IV.C (Table 4) on a
synthetic stereo clip (the paper's MPEG-7 clips are not available): per block of 50/100/200 ms,
the left block (zero-padded to all 2B-1 lags) is cross-correlated with the right block, each
right block companded as its own kernel (S_q = K_q = 32 as in P:203 where the packing's bound
allows it, else the largest Q that does; PAPER R_max, dyadic eps).  Reports per block size and
packing: xcorr throughput in input samples/s of one channel (timed: per-pair kernel companding +
the packed cross-correlations + scores), the relative-delay error rate, the cross-channel
correlation error (normalized peak rho = c_max / sqrt(E_x E_q)) and the mono/stereo decision
(mono iff the peak is at lag 0 and rho >= 0.99) against full precision, and the speed-up.
    python tools/mpeg7_stereo.py [seconds]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1201_3018_b200 import binding as pcb
from paper_1201_3018_b200 import workloads as WL

FULL, SYM, ASYM2, ASYM3 = 0, 1, 2, 3
NAMES = {FULL: "full", SYM: "sym", ASYM2: "asym2", ASYM3: "asym3"}
seconds = float(sys.argv[1]) if len(sys.argv) > 1 else 60.0
dev = torch.device("cuda")
delay = 17
clips = {"stereo": WL.stereo(seed=0, seconds=seconds, delay=delay), "mono": WL.stereo(seed=1, seconds=seconds,
                                                                                    delay=0, mono=True)}


def w_block_for(B):
    Np = B | 1
    w = 1
    while w < 3 * Np + 1:
        w *= 2
    return w


def max_q(B, pk):
    if pk == FULL:
        return 0
    Np = B | 1
    bound = {SYM: 131071, ASYM2: 67108863, ASYM3: 131071}[pk]   # dyadic-eps bounds (reading C4)
    q = 32
    while q > 0 and Np * q * q > bound:
        q -= 1
    return q


out = {"clip_seconds": seconds, "delay": delay, "rows": []}
for B in (2205, 4410, 8820):
    Wb = w_block_for(B)
    per_clip = {}
    for clip, (left, right) in clips.items():
        x, q = WL.stereo_pairs(left, right, B)
        n, L = x.shape
        X, Qd = torch.from_numpy(x).to(dev), torch.from_numpy(q).to(dev)
        ex = np.sum(x * x, axis=1)
        eq = np.sum(q * q, axis=1)
        res = {}
        for pk in (FULL, SYM, ASYM2, ASYM3):
            Q = max_q(B, pk)
            if pk != FULL and Q < 1:
                continue
            with pcb.Plan(L, B, Wb, pcb.MODE_XCORR, pk, Q, rmax_rule=pcb.RMAX_PAPER) as p:
                sc = torch.empty(n, dtype=torch.float64, device=dev)
                lag = torch.empty(n, dtype=torch.int64, device=dev)

                def step():
                    p.set_kernels(Qd, n, B)
                    p.xcorr_pairs(X, n, L, sc, lag)

                for _ in range(3):
                    step()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                steps = 10
                for _ in range(steps):
                    step()
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / steps
                s_np, l_np = sc.cpu().numpy(), lag.cpu().numpy()
            rho = s_np / np.sqrt(np.maximum(ex * eq, 1e-300))
            res[NAMES[pk]] = {"Q": Q, "ms": ms, "samples_per_s": n * B / (ms / 1e3),
                              "delay": (l_np - (B - 1)).tolist(), "rho": rho.tolist()}
        arr = {name: (np.array(r.pop("delay")), np.array(r.pop("rho"))) for name, r in res.items()}
        d_ref, rho_ref = arr["full"]
        for name, r in res.items():
            d, rho = arr[name]
            r["delay_error_rate"] = float(np.mean(d != d_ref))
            r["corr_error_rel"] = float(np.mean(np.abs(rho - rho_ref) / np.abs(rho_ref)))
            # mono/stereo decision (the paper does not define it; reading): mono iff the peak is at
            # lag 0 and the normalized cross-channel correlation is >= 0.99
            mono = (d == 0) & (rho >= 0.99)
            r["mono_stereo_correct_rate"] = float(np.mean(mono == (clip == "mono")))
            r["delay_true_rate"] = float(np.mean(d == (0 if clip == "mono" else -delay)))
        for name, r in res.items():
            r["speedup_vs_full"] = res["full"]["ms"] / r["ms"]
        per_clip[clip] = res
    out["rows"].append({"B": B, "ms_block": round(1000 * B / 44100), "W_block": Wb, "clips": per_clip})
print(json.dumps(out, indent=1))
