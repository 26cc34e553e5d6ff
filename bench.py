"""Benchmark of the packed approximate overlap-save convolution on B200 (arXiv 1201.3018).

Metric (BASELINE.json): output samples/s of the packed path vs the full-precision path on
the same GPU, plus the fraction of the FP64 FMA roofline of the hot kernel.

Default workload: BASELINE.json configs[1] ("cfg2"): L = 2^22 synthetic audio samples,
N = 512 windowed-sinc kernel, W_block = 4096, direct core.  Headline operating point:
asymmetric packing M=2 at 10 bits (Q = 511), L1 companding range (reading C3), dyadic eps
(reading C4) -- the config's >= 40 dB point.  One step = one pass of the whole hot path
(companding, packing, packed FP64 core, unpacking, dequantization, placement) over one
signal per GPU.  N GPUs: N independent cfg2 signals (seed = rank), one per rank, no
collective on the data path ("scaling": "weak").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED_FP64_TFLOPS = 34.0   # profiles/r01_fp64_peak.log: sustained DFMA, 148 SMs @ 1965 MHz
FP64_PEAK_SOURCE = "measured (tools/fp64_peak.cu, profiles/r01_fp64_peak.log); not in MEASURED_PEAKS.json"

POINTS = {
    # name: (packing, Q, rmax_rule)  -- packing codes of include/packedconv.h
    "asym2_10b": (2, 511, 1),
    "asym2_8b": (2, 127, 1),
    "asym3_8b": (3, 127, 1),
    "sym_8b": (1, 127, 1),
    "sym_6b": (1, 31, 1),
    "full": (0, 0, 0),
}
HEADLINE = "asym2_10b"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--points", default=",".join(POINTS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--L", type=int, default=0, help="override the workload length (scaling studies)")
    return ap.parse_args()


class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and "Active" == r[3 + i]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_setup(args):
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        backend = "nccl" if args.impl == "ours" else "gloo"
        if args.impl == "ours":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    elif args.impl == "ours":
        torch.cuda.set_device(0)
    return ws, rank, local


def max_over_ranks(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def workload(name, rank, L=0):
    from paper_1201_3018_b200 import workloads as WL
    if name == "cfg2":
        s, k = WL.cfg2(seed=rank, L=L or (1 << 22))
        return s, k, 4096
    if name == "cfg1":
        s, k = WL.cfg1(seed=rank)
        return s, k, 1024
    if name == "cfg5":
        s, k = WL.cfg5(seed=rank, L=1 << 24)
        return s, k, 4096
    raise SystemExit(f"unknown workload {name}")


def cpu_baseline(s, k, W_block, point, target_s=12.0):
    """The oracle as it stands, on a bounded sample of the same workload: consecutive
    blocks from block 1 until ~target_s seconds of CPU work; value = output samples/s."""
    import oracle as O
    packing, Q, rmax = POINTS[point]
    geom = O.Geometry(len(s), len(k), W_block)
    ks = O.prepare_kernel(k, geom, packing, Q, None, O.CONV, O.EPS_POW2, rmax)
    t0 = time.perf_counter()
    n = 0
    w = 1
    while time.perf_counter() - t0 < target_s and w < geom.P:
        O.process_block(s, w, geom, ks, Q)
        n += 1
        w += 1
    dt = time.perf_counter() - t0
    return {"value": n * geom.W / dt, "unit": "output samples/s", "cores": 1, "kind": "oracle",
            "sample": f"{n} consecutive overlap-save blocks ({n * geom.W} outputs) of {point} at cfg2, "
                      f"NumPy oracle single-threaded (np.convolve)"}


def run_reference(args, ws, rank):
    if rank != 0:
        return
    s, k, W_block = workload(args.workload, 0)
    import oracle as O
    packing, Q, rmax = POINTS[HEADLINE]
    geom = O.Geometry(len(s), len(k), W_block)
    ks = O.prepare_kernel(k, geom, packing, Q, None, O.CONV, O.EPS_POW2, rmax)
    blocks_per_step = 8
    for i in range(args.warmup):
        O.process_block(s, 1 + i % (geom.P - 1), geom, ks, Q)
    t0 = time.perf_counter()
    for i in range(args.steps):
        for j in range(blocks_per_step):
            O.process_block(s, 1 + (i * blocks_per_step + j) % (geom.P - 1), geom, ks, Q)
    dt = time.perf_counter() - t0
    outs = args.steps * blocks_per_step * geom.W
    v = outs / dt
    line = {"metric": "output samples/s, packed vs full-precision conv", "value": v, "unit": "output samples/s",
            "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, "point": HEADLINE, "L": len(s), "N": len(k), "W_block": W_block,
                       "step": f"{blocks_per_step} overlap-save blocks (bounded sample of the workload)"},
            "cpu_baseline": {"value": v, "unit": "output samples/s", "cores": 1, "kind": "oracle",
                             "sample": f"{blocks_per_step} blocks per step, NumPy oracle single-threaded"},
            "e2e": {"value": v, "unit": "output samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def run_ours(args, ws, rank, local):
    import torch
    from paper_1201_3018_b200 import binding as pcb

    dev = torch.device("cuda", local)
    s, k, W_block = workload(args.workload, rank, args.L)
    L, N = len(s), len(k)
    L_out = L + N - 1
    n_buf = max(2, -(-256 * (1 << 20) // (16 * L)))     # rotating buffers: > 126 MB L2 in total
    S = [torch.from_numpy(s).to(dev) for _ in range(n_buf)]
    R = [torch.empty(L_out, dtype=torch.float64, device=dev) for _ in range(n_buf)]
    k_d = torch.from_numpy(k).to(dev)
    stream = torch.cuda.current_stream(dev)
    results = {}
    outputs = {}
    sampler_summary = None
    for name in args.points.split(","):
        packing, Q, rmax = POINTS[name]
        plan = pcb.Plan(L, N, W_block, pcb.MODE_CONV, packing, Q, rmax_rule=rmax)
        plan.set_kernel(k_d)
        info = plan.info()
        for i in range(args.warmup):
            plan.execute(S[i % n_buf], R[i % n_buf])
        torch.cuda.synchronize(dev)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sampler = ClockSampler(local) if name == HEADLINE else None
        if sampler:
            sampler.__enter__()
            time.sleep(0.3)
        barrier(ws)
        torch.cuda.synchronize(dev)
        t0.record(stream)
        for i in range(args.steps):
            ev[i][0].record(stream)
            plan.execute(S[i % n_buf], R[i % n_buf])
            ev[i][1].record(stream)
        t1.record(stream)
        torch.cuda.synchronize(dev)
        barrier(ws)
        if sampler:
            # keep sampling under load long enough to see the clocks (untimed repeats)
            t_end = time.time() + 1.0
            while time.time() < t_end:
                for i in range(50):
                    plan.execute(S[i % n_buf], R[i % n_buf])
                torch.cuda.synchronize(dev)
            sampler.__exit__()
            sampler_summary = sampler.summary()
        ms = t0.elapsed_time(t1)
        ms = max_over_ranks(ms, ws)
        kern_ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
        # algorithmic FP64 work of the core per launch: sum over blocks of M_out * K FMAs
        Np, W, P, K = info["Np"], info["W"], info["P"], info["taps"]
        if packing == 0:
            m_first, m_rest = W + Np - 1, W
        elif packing == 1:
            m_first, m_rest = (W + Np - 1) // 2, W // 2 + 1
        else:
            M = 2 if packing == 2 else 3
            m_first, m_rest = -(-(W + Np - 1) // M), -(-W // M)
        fma = (m_first + (P - 1) * m_rest) * K
        results[name] = {"ms_per_step": ms / args.steps, "kernel_ms": kern_ms,
                         "value": ws * L_out * args.steps / (ms / 1e3),
                         "fp64_tflops": 2.0 * fma / (kern_ms / 1e3) / 1e12, "fma_per_output": fma / L_out,
                         "R_max": info["R_max"], "Q": Q, "bound_ok": info["bound_ok"], "tile": info["core_tile"]}
        outputs[name] = R[(args.steps - 1) % n_buf].clone()
        if name == HEADLINE:
            # end to end through the C ABI with HOST buffers (pinned): H2D + run + D2H per step
            sh = torch.from_numpy(s).pin_memory()
            rh = torch.empty(L_out, dtype=torch.float64).pin_memory()
            for i in range(2):
                plan.execute_host(sh, rh)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n_e2e = max(3, min(args.steps, 20))
            barrier(ws)
            torch.cuda.synchronize(dev)
            e0.record(stream)
            for i in range(n_e2e):
                plan.execute_host(sh, rh)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            e_ms = max_over_ranks(e0.elapsed_time(e1), ws)
            results[name]["e2e"] = {"value": ws * L_out * n_e2e / (e_ms / 1e3), "unit": "output samples/s",
                                    "h2d_bytes_per_step": 8 * L, "d2h_bytes_per_step": 8 * L_out,
                                    "steps": n_e2e}
        plan.close()
    # accuracy of every point against the GPU full-precision path (same input)
    if "full" in outputs:
        ref = outputs["full"].double()
        for name, out in outputs.items():
            if name == "full":
                continue
            err = torch.sum((ref - out) ** 2).item()
            results[name]["snr_db_vs_full"] = 10 * np.log10(torch.sum(ref * ref).item() / err) if err > 0 else None
    if rank != 0:
        return
    h = results[HEADLINE]
    full = results.get("full")
    traffic, traffic_src = None, None
    prof = os.path.join(ROOT, "profiles", "r01_ncu_cfg2.json")
    kname = f"pc_persist_kernel<2, {h['tile']}>"
    if args.workload == "cfg2" and os.path.exists(prof):
        for rec in json.load(open(prof)).get("ncu_full", []):
            if kname in rec["kernel"]:
                rd = float(rec["dram__bytes_read.sum"].split()[0]) * (1e6 if "Mbyte" in rec["dram__bytes_read.sum"] else 1e3)
                wr = rec["dram__bytes_write.sum"].split()
                wr = float(wr[0]) * (1e6 if wr[1] == "Mbyte" else 1e3 if wr[1] == "Kbyte" else 1.0)
                traffic, traffic_src = rd + wr, "profiles/r01_ncu_cfg2.json (ncu --set full, one launch)"
    roof = {"bound": "alu", "achieved": h["fp64_tflops"], "peak": MEASURED_FP64_TFLOPS, "unit": "TFLOP/s",
            "frac": h["fp64_tflops"] / MEASURED_FP64_TFLOPS, "traffic": traffic, "traffic_unit": "bytes/launch",
            "traffic_source": traffic_src, "algorithmic_bytes": 8 * (L + L_out),
            "kernel": kname, "peak_source": FP64_PEAK_SOURCE,
            "algorithmic": "FP64 FMAs of the packed core: sum over blocks of M_out * N' (2 flop each)"}
    line = {
        "metric": "output samples/s, packed vs full-precision conv, 1/2/4/8 B200; % FP64/HBM peak",
        "value": h["value"], "unit": "output samples/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": h["ms_per_step"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "L": L, "N": N, "W_block": W_block, "point": HEADLINE,
                   "packing": "asym2", "bits": 10, "Q": 511, "rmax_rule": "l1", "eps": "pow2",
                   "l2": f"{n_buf} rotating input/output buffer pairs ({n_buf * 16 * L >> 20} MiB) > 126 MB L2",
                   "parallelism": f"{ws} independent signals (one per GPU), no collective"},
        "gpu_launches": args.steps,
        "roofline": roof,
        "e2e": h.get("e2e"),
        "packed_vs_full": (h["value"] / full["value"]) if full else None,
        "full_precision": full,
        "points": results,
        "clocks": sampler_summary,
    }
    if ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(s, k, W_block, HEADLINE)
    print(json.dumps(line))


def main():
    args = parse()
    ws, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, ws, rank)
    else:
        run_ours(args, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
