"""throughput of every packing vs kernel length N (Fig. 3a/3b setting,
W_block = 32 * 2^10) and vs block size at N = 800 (Fig. 2 setting), on the §IV.A workload
(input and kernel i.i.d. uniform [-128, 128], L = 8192 * 2^10), with the ranking
predicted by Table 1's time-domain FLOP model next to the measured one.

Q = S_q = K_q = 16 where the packing's bound (dyadic eps, L1 companding range) allows
it, else the largest Q that does (found through the library's own bound check).  Runs only
the product path (C ABI); prints one JSON document.
    python tools/sweep_n.py [--quick]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1201_3018_b200 import binding as pcb

FULL, SYM, ASYM2, ASYM3 = 0, 1, 2, 3
NAMES = {FULL: "full", SYM: "sym", ASYM2: "asym2", ASYM3: "asym3"}
TABLE1 = {FULL: lambda n: 4 * n * n, SYM: lambda n: n * n + n, ASYM2: lambda n: 2.5 * n * n - n,
          ASYM3: lambda n: 2 * n * n - 2.0 / 3.0 * n}    # time-domain FLOP per 2N outputs
dev = torch.device("cuda")
quick = "--quick" in sys.argv
L = (1 << 20) if quick else 8192 * 1024
rng = np.random.default_rng(0)
s = rng.uniform(-128.0, 128.0, L)
S = torch.from_numpy(s).to(dev)


def feasible(N, W_block, pk, Q, k_d):
    try:
        with pcb.Plan(L, N, W_block, pcb.MODE_CONV, pk, Q, rmax_rule=pcb.RMAX_L1, bound_policy=0) as p:
            p.set_kernel(k_d)
        return True
    except pcb.PcError:
        return False


def pick_q(N, W_block, pk, k_d):
    if pk == FULL:
        return 0
    if feasible(N, W_block, pk, 16, k_d):
        return 16
    lo, hi = 0, 16                     # largest feasible Q < 16 (R grows with Q)
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if feasible(N, W_block, pk, mid, k_d):
            lo = mid
        else:
            hi = mid
    return lo


def run(N, W_block, pk, Q, k_d, steps=10):
    with pcb.Plan(L, N, W_block, pcb.MODE_CONV, pk, Q, rmax_rule=pcb.RMAX_L1) as p:
        p.set_kernel(k_d)
        R = torch.empty(L + N - 1, dtype=torch.float64, device=dev)
        for _ in range(3):
            p.execute(S, R)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(steps):
            p.execute(S, R)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        return ms, R


out = {"workload": f"uniform [-128,128] input and kernel, L = {L}", "q_rule": "16 if feasible (L1 range, dyadic eps)",
       "vs_N": [], "vs_W_block": []}
Ns = [32, 64, 128, 256, 512, 1024, 2048, 4096, 8192] if not quick else [64, 512, 4096]
for N in Ns:
    k = rng.uniform(-128.0, 128.0, N)
    k_d = torch.from_numpy(k).to(dev)
    row = {"N": N, "W_block": 32768, "modes": {}}
    ref = None
    for pk in (FULL, SYM, ASYM2, ASYM3):
        Q = pick_q(N, 32768, pk, k_d)
        if pk != FULL and Q < 1:
            row["modes"][NAMES[pk]] = {"feasible": False}
            continue
        ms, R = run(N, 32768, pk, Q, k_d)
        rec = {"Q": Q, "us": round(ms * 1e3, 2), "samples_per_s": (L + N - 1) / (ms / 1e3)}
        if pk == FULL:
            ref = R.clone()
        else:
            err = torch.sum((ref - R) ** 2).item()
            rec["snr_db"] = round(10 * np.log10(torch.sum(ref * ref).item() / err), 2) if err > 0 else None
        row["modes"][NAMES[pk]] = rec
    full_us = row["modes"]["full"]["us"]
    live = [m for m in (SYM, ASYM2, ASYM3) if row["modes"][NAMES[m]].get("us")]
    for m in live:
        row["modes"][NAMES[m]]["speedup_vs_full"] = round(full_us / row["modes"][NAMES[m]]["us"], 3)
        row["modes"][NAMES[m]]["table1_flop_ratio"] = round(TABLE1[FULL](N) / TABLE1[m](N), 3)
    row["measured_rank"] = sorted([NAMES[m] for m in live], key=lambda n: row["modes"][n]["us"])
    row["table1_rank"] = sorted([NAMES[m] for m in live], key=lambda n: TABLE1[[k_ for k_, v in NAMES.items() if v == n][0]](N))
    out["vs_N"].append(row)

N = 800
k = rng.uniform(-128.0, 128.0, N)
k_d = torch.from_numpy(k).to(dev)
for Wb in ([4096, 8192, 16384, 32768, 65536] if not quick else [4096, 32768]):
    row = {"N": N, "W_block": Wb, "modes": {}}
    for pk in (FULL, SYM, ASYM2, ASYM3):
        Q = pick_q(N, Wb, pk, k_d)
        if pk != FULL and Q < 1:
            row["modes"][NAMES[pk]] = {"feasible": False}
            continue
        ms, _ = run(N, Wb, pk, Q, k_d)
        row["modes"][NAMES[pk]] = {"Q": Q, "us": round(ms * 1e3, 2), "samples_per_s": (L + N - 1) / (ms / 1e3)}
    out["vs_W_block"].append(row)
print(json.dumps(out, indent=1))
