"""Benchmark of the packed approximate overlap-save convolution on B200 (arXiv 1201.3018).

Metric (BASELINE.json): output samples/s of the packed path vs the full-precision path on
the same GPU, plus the fraction of the FP64 (direct core) / HBM (FFT core) roofline of the
hot kernel.

Headline workload: BASELINE.json configs[1] ("cfg2"): synthetic audio, N = 512 windowed-sinc
kernel, W_block = 4096, direct core.  Operating point: asymmetric packing M=2 at 10 bits
(Q = 511), L1 companding range (reading C3), dyadic eps (reading C4) -- the config's >= 40 dB
point.  One step = one pass of the whole hot path (companding, packing, packed FP64 core,
unpacking, dequantization, placement).  N GPUs (SURVEY §8(e), B:north_star): ONE signal of
N * 2^22 samples split by overlap-save block range -- every rank generates the same global
signal, keeps only its shard (conv_shard_range: its blocks' input plus the N'+1-sample halo)
and runs conv_execute_blocks on it; no collective on the data path ("scaling": "weak", so
N = 1 is the single 2^22-sample signal).

Sub-records of the default run (the other BASELINE.json configs):
  cfg3  FFT core, L = 2^24, block-range split at the stated L (strong scaling)
  cfg5  SNR-adaptive 40 dB, L = 2^26, block-range split (conv_adapt_blocks + conv_execute_blocks)
  cfg4  cross-correlation database sharded by signal (a bounded database: --cfg4-signals per
        rank), the timed step including the NCCL all-gather of the per-rank winners
--workload cfgX makes X the headline (cfg4 then at its full 1024 signals unless --signals).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload cfgX]

--gpus N > 1 without torchrun's environment re-launches itself through torch.distributed.run
(one process per GPU, NCCL).  A one-rank NCCL group is initialised at N = 1 as well.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED_FP64_TFLOPS = 34.0   # profiles/r01_fp64_peak.log: sustained DFMA, 148 SMs @ 1965 MHz
FP64_PEAK_SOURCE = "measured (tools/fp64_peak.cu, profiles/r01_fp64_peak.log); not in MEASURED_PEAKS.json"
MEASURED_DMMA_TFLOPS = 37.1   # profiles/r01_dmma_peak.log: FP64 tensor cores (mma.sync m8n8k4 f64)
DMMA_PEAK_SOURCE = ("measured (tools/dmma_peak.cu, profiles/r01_dmma_peak.log: 18.56 T DMMA-FMA/s); "
                    "not in MEASURED_PEAKS.json")
HBM_GBS_FALLBACK = 6540.2


def hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:                                   # noqa: BLE001
        return HBM_GBS_FALLBACK, "round-1 copy of MEASURED_PEAKS.json hbm_gbs"


METRIC = "output samples/s, packed vs full-precision conv, 1/2/4/8 B200; % FP64/HBM peak"   # BASELINE.json
FULL, SYM, ASYM2, ASYM3, ADAPT = 0, 1, 2, 3, 4
DIRECT, FFT = 0, 1
WARN = {"bound_policy": 1}
# workload -> (W_block, points {name: (packing, Q|floor, rmax_rule, core[, extra conv_opts])}, headline, full point)
WORKLOADS = {
    "cfg1": (1024, {"asym2_9b": (ASYM2, 255, 0, DIRECT), "asym2_8b": (ASYM2, 127, 0, DIRECT),
                    "sym_q44": (SYM, 44, 0, DIRECT), "full": (FULL, 0, 0, DIRECT)}, "asym2_9b", "full"),
    "cfg2": (4096, {"asym2_10b": (ASYM2, 511, 1, DIRECT), "asym2_8b": (ASYM2, 127, 1, DIRECT),
                    "asym3_8b": (ASYM3, 127, 1, DIRECT), "sym_8b": (SYM, 127, 1, DIRECT),
                    "sym_6b": (SYM, 31, 1, DIRECT), "full": (FULL, 0, 0, DIRECT)}, "asym2_10b", "full"),
    # cfg3: asym2 Q = 191 is the largest asym2 point the FFT backend validation accepts under
    # STRICT at this geometry; 9 bits (Q = 255) fails it on worst-case operands and
    # runs under WARN with the residual monitor.  full_fft32k = the configured full-precision core
    # (the block's 32768-point transform); full_fft = the fair circular transform of the cost model.
    "cfg3": (16384, {"asym2_q191_fft": (ASYM2, 191, 1, FFT), "asym2_9b_fft": (ASYM2, 255, 1, FFT, WARN),
                     "sym_q8_fft": (SYM, 8, 1, FFT), "full_fft32k": (FULL, 0, 0, FFT, {"fft_n": 16384}),
                     "full_fft": (FULL, 0, 0, FFT),
                     "asym2_9b_direct": (ASYM2, 255, 1, DIRECT), "full_direct": (FULL, 0, 0, DIRECT)},
             "asym2_q191_fft", "full_fft32k"),
    "cfg4": (32768, {"asym2_8b": (ASYM2, 127, 1, DIRECT), "sym_q7": (SYM, 7, 1, DIRECT),
                     "full": (FULL, 0, 0, DIRECT)}, "asym2_8b", "full"),
    "cfg5": (4096, {"adapt_40db": (ADAPT, 40.0, 1, DIRECT), "adapt_50db": (ADAPT, 50.0, 1, DIRECT),
                    "adapt_60db": (ADAPT, 60.0, 1, DIRECT), "full": (FULL, 0, 0, DIRECT)}, "adapt_40db", "full"),
}
SUB_POINTS = {"cfg3": ["asym2_q191_fft", "asym2_9b_fft", "full_fft32k", "full_fft"],
              "cfg5": ["adapt_40db", "full"], "cfg4": ["asym2_8b", "full"]}
BASE_L = {"cfg1": 65536, "cfg2": 1 << 22, "cfg3": 1 << 24, "cfg5": 1 << 26}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS))
    ap.add_argument("--points", default="", help="comma-separated subset of the headline workload's points")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sub", action="store_true", help="skip the cfg3/cfg5/cfg4 sub-records")
    ap.add_argument("--cfg4-signals", type=int, default=32, help="cfg4 sub-record: database signals per rank")
    ap.add_argument("--L", type=int, default=0, help="override the headline signal length (per rank for cfg2)")
    ap.add_argument("--signals", type=int, default=0, help="cfg4 headline: database signals in total (default 1024)")
    ap.add_argument("--force-warps", type=int, default=0, help="diagnostics: consumer warps per job")
    ap.add_argument("--opt", action="append", default=[], help="diagnostics: a named conv_opts field as name=v")
    ap.add_argument("--N", type=int, default=0, help="diagnostics: override the kernel length (cfg1/cfg2)")
    ap.add_argument("--exec", default="fused", choices=["fused", "perblock"], help="diagnostics: execution form")
    ap.add_argument("--graph", type=int, default=1,
                    help="1 (default): the K timed steps are captured in one CUDA graph and replayed (every "
                         "launch of every step runs; no host submission gaps); 0: launched back to back")
    return ap.parse_args()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch(args):
    """--gpus N > 1 outside torchrun: one process per GPU through torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


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
            except Exception:                           # noqa: BLE001
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


# ------------------------------------------------------------------------------ process group
class Dist:
    """One process per GPU; a process group is always initialised (a one-rank NCCL group at N = 1,
    so the NCCL path of the score gather runs on a single-GPU box too)."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist
        if "WORLD_SIZE" not in os.environ:
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), RANK="0", WORLD_SIZE="1",
                              LOCAL_RANK="0")
        self.ws = int(os.environ["WORLD_SIZE"])
        self.rank = int(os.environ["RANK"])
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.gpu = args.impl == "ours"
        self.backend = "nccl" if self.gpu else "gloo"
        if self.gpu:
            torch.cuda.set_device(self.local)
            dist.init_process_group(self.backend, device_id=torch.device("cuda", self.local))
        else:
            dist.init_process_group(self.backend)
        self.dist = dist

    def _t(self, vals):
        import torch
        return torch.tensor(vals, dtype=torch.float64, device="cuda" if self.gpu else "cpu")

    def max(self, x):
        t = self._t([x])
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, *xs):
        t = self._t(list(xs))
        self.dist.all_reduce(t)
        return [float(v) for v in t.cpu().tolist()]

    def bcast(self, x):
        t = self._t([x])
        self.dist.broadcast(t, 0)
        return float(t.item())

    def barrier(self):
        if self.gpu:
            import torch
            self.dist.barrier(device_ids=[self.local])
            torch.cuda.synchronize()
        else:
            self.dist.barrier()

    def close(self):
        self.dist.destroy_process_group()


# ------------------------------------------------------------------------------ workloads
def gen(name, L, N=0):
    from paper_1201_3018_b200 import workloads as WL
    if name == "cfg1":
        return WL.cfg1(seed=0, L=L, N=N or 64)
    if name == "cfg2":
        return WL.cfg2(seed=0, L=L, N=N or 512)
    if name == "cfg3":
        return WL.cfg3(seed=0, L=L)
    return WL.cfg5(seed=0, L=L)


def _cfg4_sig(i):
    from paper_1201_3018_b200 import workloads as WL
    return WL.cfg4_signal(i)


def core_fma_blocks(info, packing, b0, b1, blocks=None):
    """Algorithmic FP64 FMAs of the packed core over blocks [b0, b1) (or a list): per block
    M_out * K, K = N' (or ceil(N'/2) for symmetric packing)."""
    Np, W = info["Np"], info["W"]
    K = (Np + 1) // 2 if packing == SYM else Np
    if packing == FULL:
        m_first, m_rest = W + Np - 1, W
    elif packing == SYM:
        m_first, m_rest = (W + Np - 1) // 2, W // 2 + 1
    else:
        M = 2 if packing == ASYM2 else 3
        m_first, m_rest = -(-(W + Np - 1) // M), -(-W // M)
    if blocks is not None:
        return sum(m_first if w == 0 else m_rest for w in blocks) * K
    n = b1 - b0
    return ((m_first if b0 == 0 else m_rest) + (n - 1) * m_rest) * K if n > 0 else 0


def make_opts(pcb, args, rmax, core, extra):
    opts = pcb.opts_default(rmax_rule=rmax, core=core, exec=0 if args.exec == "fused" else 1)
    opts.parts_per_job = args.force_warps
    # The opt-in launch overlap (a persistent launch's pipeline fill may run during the preceding
    # launch's tail, host-checked not to read what that launch writes): safe here because this
    # process's streams carry only this library's launches -- no foreign kernel with its own
    # programmatic trigger can sit between two of them (include/packedconv.h, early_fill).
    opts.early_fill = 1
    for f, v in extra.items():
        setattr(opts, f, v)
    for kv in args.opt:
        f, v = kv.split("=")
        setattr(opts, f, int(v))
    return opts


def time_steps(step, args, D, dev, stream, use_graph, sampler=None):
    """W untimed warm-up steps, then EXACTLY K steps bracketed by a barrier + synchronize on both
    sides, timed with CUDA events on the launching stream (optionally replayed from one CUDA
    graph); returns (this rank's ms, max over ranks ms)."""
    import torch
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize(dev)
    graph = None
    if use_graph:                                      # K steps replayed as one graph (no host launch gaps)
        gs = torch.cuda.Stream(dev)
        gs.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(gs):
            with torch.cuda.graph(graph, stream=gs):
                for i in range(args.steps):
                    step(i)
        stream.wait_stream(gs)
        graph.replay()
        torch.cuda.synchronize(dev)
    if sampler:
        sampler.__enter__()
        time.sleep(0.3)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    D.barrier()
    torch.cuda.synchronize(dev)
    t0.record(stream)
    if graph is not None:
        graph.replay()
    else:
        for i in range(args.steps):
            step(i)
    t1.record(stream)
    torch.cuda.synchronize(dev)
    D.barrier()
    if sampler:                                        # keep the GPU busy while the sampler reads clocks
        t_end = time.time() + 1.0
        while time.time() < t_end:
            if graph is not None:
                graph.replay()
            else:
                for i in range(args.steps):
                    step(i)
            torch.cuda.synchronize(dev)
        sampler.__exit__()
    ms = t0.elapsed_time(t1)
    return ms, D.max(ms)


# ------------------------------------------------------------------------------ block-range split
def measure_split(name, sel, head, args, D, dev, L_global, clocks=False, N_override=0):
    """One signal of L_global samples split by overlap-save block range over the ranks
    (conv_shard_range + conv_execute_blocks / conv_adapt_blocks); every point in `sel`."""
    import torch
    from paper_1201_3018_b200 import binding as pcb
    W_block, points, _, full_pt = WORKLOADS[name]
    x, k = gen(name, L_global, N_override)
    L, N = len(x), len(k)
    L_out = L + N - 1
    sh = pcb.shard_range(L, N, W_block, pcb.MODE_CONV, D.rank, D.ws)
    b0, b1, i0, i1, o0, o1 = (sh[f] for f in ("block_begin", "block_end", "in_begin", "in_end", "out_begin", "out_end"))
    xs = np.ascontiguousarray(x[i0:i1])
    n_out = max(1, o1 - o0)
    per_buf = 8 * (len(xs) + n_out)
    n_buf = max(2, -(-256 * (1 << 20) // per_buf))    # rotating buffers: > 126 MB L2 between steps
    S = [torch.from_numpy(xs).to(dev) for _ in range(n_buf)]
    R = [torch.empty(n_out, dtype=torch.float64, device=dev) for _ in range(n_buf)]
    k_d = torch.from_numpy(k).to(dev)
    stream = torch.cuda.current_stream(dev)
    results, outputs, sampler_summary = {}, {}, None
    for pname in sel:
        packing, Q, rmax, core = points[pname][:4]
        extra = points[pname][4] if len(points[pname]) > 4 else {}
        adaptive = packing == ADAPT
        opts = make_opts(pcb, args, rmax, core, extra)
        plan = pcb.Plan(L, N, W_block, pcb.MODE_CONV, packing, 0 if adaptive else Q, opts=opts)
        plan.set_kernel(k_d)
        info = plan.info()
        calib = 0.0
        if adaptive:
            # §IV.D: the SNR model calibrated once at S_q = K_q = 8 on rank 0's shard (a
            # plan of the shard's length), broadcast so every rank decides with the same offset
            if D.rank == 0:
                with pcb.Plan(len(xs), N, W_block, pcb.MODE_CONV, packing, 0, opts=opts) as pc_:
                    calib, _, _ = pc_.snr_calibrate(S[0], k_d, 8)
            calib = D.bcast(calib)

        def step(i, plan=plan, adaptive=adaptive, Q=Q, calib=calib):
            j = i % n_buf
            if adaptive:
                plan.adapt_blocks(S[j], i0, b0, b1, Q, calib)
            plan.execute_blocks(S[j], i0, R[j], o0, b0, b1)

        sampler = ClockSampler(D.local) if (clocks and pname == head) else None
        ms, ms_max = time_steps(step, args, D, dev, stream, args.graph == 1, sampler)
        if sampler:
            sampler_summary = sampler.summary()
        kern_ms = ms / args.steps
        if adaptive:                                   # the blocks each packing ran on this shard
            dec = plan.adapt_blocks(S[(args.steps - 1) % n_buf], i0, b0, b1, Q, calib, want=True) or []
            fma = sum(core_fma_blocks(info, pk, 0, 0, [b0 + w for w, d in enumerate(dec) if d[0] == pk])
                      for pk in (FULL, SYM, ASYM2))
            counts = D.sum(*[sum(1 for d in dec if d[0] == pk) for pk in (FULL, SYM, ASYM2)])
        else:
            fma = core_fma_blocks(info, packing, b0, b1)
        fma_all = D.sum(fma)[0]
        rec = {"ms_per_step": ms_max / args.steps, "kernel_ms_rank0": kern_ms,
               "value": L_out * args.steps / (ms_max / 1e3), "R_max": info["R_max"], "Q": Q,
               "bound_ok": info["bound_ok"], "tile": info["core_tile"], "fft_n": info["fft_n"],
               "core": "fft" if core == FFT else "direct", "exec": info["exec_used"], "cuda_graph": args.graph == 1,
               "core_mma": info["core_mma"]}
        if core == DIRECT:                             # per GPU: all ranks' FMAs over the max step time
            rec["fp64_tflops"] = 2.0 * fma_all / D.ws / (ms_max / args.steps / 1e3) / 1e12
            rec["fma_per_output"] = fma_all / L_out
        else:
            res, _ = plan.residual()
            rec["fft_residual_lsb"] = D.max(res)
            rec["backend_ok"], rec["backend_resid_lsb"], rec["u_sys_cal"] = (info["backend_ok"], info["backend_resid"],
                                                                             info["u_sys_cal"])
            rec["hbm_gbs_algorithmic"] = 8 * (L + L_out) / D.ws / (ms_max / args.steps / 1e3) / 1e9
        if extra.get("bound_policy") == 1:
            rec["bound_policy"] = "WARN (fails the STRICT backend validation; residual monitor reported)"
        if adaptive:
            rec["blocks_per_packing"] = dict(zip(("full", "sym", "asym2"), [int(c) for c in counts]))
            rec["calib_offset_db"] = calib
        results[pname] = rec
        outputs[pname] = R[(args.steps - 1) % n_buf][:o1 - o0].clone()
        if pname == head and not adaptive:             # e2e: pinned host slice through the C ABI
            sh_h = torch.from_numpy(xs).pin_memory()
            rh = torch.empty(n_out, dtype=torch.float64).pin_memory()
            for _ in range(2):
                plan.execute_host_blocks(sh_h, i0, rh, o0, b0, b1)
            n_e2e = max(3, min(args.steps, 20))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            D.barrier()
            e0.record(stream)
            for _ in range(n_e2e):
                plan.execute_host_blocks(sh_h, i0, rh, o0, b0, b1)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            e_ms = D.max(e0.elapsed_time(e1))
            rec["e2e"] = {"value": L_out * n_e2e / (e_ms / 1e3), "unit": "output samples/s",
                          "h2d_bytes_per_step": int(8 * L), "d2h_bytes_per_step": int(8 * L_out), "steps": n_e2e,
                          "api": "conv_execute_host_blocks (pinned host shard in, host outputs back)"}
        plan.close()
    if full_pt in outputs:                             # SNR vs full precision over all ranks' outputs
        ref = outputs[full_pt]
        for pname, out in outputs.items():
            if pname == full_pt or points[pname][0] == FULL:
                continue
            sig, err = D.sum(torch.sum(ref * ref).item(), torch.sum((ref - out) ** 2).item())
            results[pname]["snr_db_vs_full"] = 10 * math.log10(sig / err) if err > 0 else None
    meta = {"L": L, "N": N, "W_block": W_block, "n_buf": n_buf, "per_buf": per_buf,
            "shard_rank0": {"blocks": [b0, b1], "input": [i0, i1], "outputs": [o0, o1]}}
    return results, sampler_summary, meta, (x, k)


# ------------------------------------------------------------------------------ cfg4: signal shards
def measure_cfg4(sel, head, args, D, dev, n_total, clocks=False):
    """Database signals sharded over ranks: per rank conv_xcorr_max over its signals, then the
    world's winner through gather_best_match (conv_best_match on each rank, NCCL all-gather of one
    candidate per rank, conv_best_match again) -- all inside the timed step."""
    import multiprocessing as mp

    import torch
    from paper_1201_3018_b200 import binding as pcb
    from paper_1201_3018_b200 import distributed as PD
    from paper_1201_3018_b200 import workloads as WL
    W_block, points, _, _ = WORKLOADS["cfg4"]
    a, b = PD.signal_range(n_total, D.rank, D.ws)
    with mp.get_context("fork").Pool(min(16, os.cpu_count() or 1)) as pool:
        sigs = pool.map(_cfg4_sig, range(a, b))
    q, i_true, off_true = WL.cfg4_query(seed=0, n_signals=n_total)
    X = torch.from_numpy(np.stack(sigs)).to(dev)
    nsig, L = X.shape
    N = len(q)
    q_d = torch.from_numpy(q).to(dev)
    stream = torch.cuda.current_stream(dev)
    results, sampler_summary = {}, None
    for pname in sel:
        packing, Q, rmax, core = points[pname][:4]
        opts = make_opts(pcb, args, rmax, core, {})
        plan = pcb.Plan(L, N, W_block, pcb.MODE_XCORR, packing, Q, opts=opts)
        plan.set_kernel(q_d)
        info = plan.info()
        score = torch.empty(nsig, dtype=torch.float64, device=dev)
        lag = torch.empty(nsig, dtype=torch.int64, device=dev)
        box = {}

        def step(i, plan=plan, score=score, lag=lag, box=box):
            plan.xcorr_max(X, nsig, L, score, lag)
            box["best"] = PD.gather_best_match(score, lag, a)

        sampler = ClockSampler(D.local) if (clocks and pname == head) else None
        ms, ms_max = time_steps(step, args, D, dev, stream, False, sampler)
        if sampler:
            sampler_summary = sampler.summary()
        fma_all = D.sum(core_fma_blocks(info, packing, 0, info["P"]) * nsig)[0]
        L_out = (L - N + 1) * n_total
        results[pname] = {"ms_per_step": ms_max / args.steps, "kernel_ms_rank0": ms / args.steps,
                          "value": L_out * args.steps / (ms_max / 1e3), "Q": Q, "R_max": info["R_max"],
                          "bound_ok": info["bound_ok"], "core_mma": info["core_mma"], "exec": info["exec_used"],
                          "tile": info["core_tile"],
                          "fp64_tflops": 2.0 * fma_all / D.ws / (ms_max / args.steps / 1e3) / 1e12,
                          "best_match": PD.best_match_tuple(box["best"]), "query_source": [i_true, off_true]}
        plan.close()
    meta = {"L": L, "N": N, "W_block": W_block, "signals_total": n_total, "signals_per_rank": nsig,
            "gather": "conv_best_match per rank + NCCL all_gather_into_tensor (3 doubles/rank) + conv_best_match"}
    return results, sampler_summary, meta


# ------------------------------------------------------------------------------ CPU baselines
def cpu_baseline(s, k, W_block, point, target_s=10.0):
    """The oracle as it stands (single-threaded NumPy), on a bounded sample of the same workload:
    consecutive overlap-save blocks from block 1 for ~target_s seconds; value = output samples/s.
    Both the packed point and full precision (BASELINE.md §3, P:153's single-thread method)."""
    import oracle as O
    packing, Q, rmax = point[:3]
    if packing not in (FULL, SYM, ASYM2, ASYM3):
        packing, Q, rmax = ASYM2, 535, 1
    geom = O.Geometry(len(s), len(k), W_block)

    def rate(pk, q, rm, t_s):
        ks = O.prepare_kernel(k, geom, pk, q, None, O.CONV, O.EPS_POW2, rm)
        t0 = time.perf_counter()
        n, w = 0, 1
        while time.perf_counter() - t0 < t_s and w < geom.P:
            O.process_block(s, w, geom, ks, q)
            n += 1
            w += 1
        return n * geom.W / (time.perf_counter() - t0), n

    v, n = rate(packing, Q, rmax, target_s)
    vf, nf = rate(FULL, 0, 0, target_s / 2)
    return {"value": v, "unit": "output samples/s", "cores": 1, "kind": "oracle",
            "sample": f"{n} consecutive overlap-save blocks ({n * geom.W} outputs), NumPy oracle single-threaded "
                      f"(np.convolve per block)",
            "full_precision": {"value": vf, "unit": "output samples/s",
                               "sample": f"{nf} blocks, the same oracle at full precision"},
            "packed_vs_full_cpu": v / vf,
            "paper_cpu_packed_vs_full": "+52%..+175% (P:181, P:199, P:212; i5 540M, IPP, single thread)"}


_CPU_STATE = {}


def _cpu_worker(args_):
    import oracle as O
    w0, w1, target_s = args_
    st = _CPU_STATE
    t0 = time.perf_counter()
    n = 0
    for w in range(w0, w1):
        if time.perf_counter() - t0 >= target_s:
            break
        O.process_block(st["s"], w, st["geom"], st["ks"], st["Q"])
        n += 1
    return n, time.perf_counter() - t0


def cpu_baseline_all_cores(s, k, W_block, point, target_s=6.0):
    """The same oracle, one process per host core over disjoint block ranges (blocks are
    independent; numerics unchanged), ~target_s seconds each."""
    import multiprocessing as mp

    import oracle as O
    packing, Q, rmax = point[:3]
    if packing not in (FULL, SYM, ASYM2, ASYM3):
        packing, Q, rmax = ASYM2, 535, 1
    geom = O.Geometry(len(s), len(k), W_block)
    ks = O.prepare_kernel(k, geom, packing, Q, None, O.CONV, O.EPS_POW2, rmax)
    _CPU_STATE.update(s=s, geom=geom, ks=ks, Q=Q)
    nproc = os.cpu_count() or 1
    P = geom.P
    ranges = [(1 + (P - 1) * i // nproc, 1 + (P - 1) * (i + 1) // nproc, target_s) for i in range(nproc)]
    with mp.get_context("fork").Pool(nproc) as pool:
        res = pool.map(_cpu_worker, ranges)
    n = sum(r[0] for r in res)
    dt = max(r[1] for r in res)
    return {"value": n * geom.W / dt, "unit": "output samples/s", "cores": nproc, "kind": "oracle",
            "sample": f"{n} overlap-save blocks in {nproc} processes (disjoint block ranges, ~{target_s:.0f} s each), "
                      f"NumPy oracle"}


# ------------------------------------------------------------------------------ reference arm
def run_reference(args, D):
    """The tier's reference arm: the CPU oracle as it stands, rank 0 only, on the headline's
    config / metric / unit; each step a bounded sample (8 overlap-save blocks) of the workload."""
    if D.rank != 0:
        return
    name = args.workload if args.workload != "cfg4" else "cfg2"
    W_block, points, head, _ = WORKLOADS[name]
    s, k = gen(name, args.L or BASE_L[name], args.N)
    import oracle as O
    packing, Q, rmax = points[head][:3]
    if packing not in (FULL, SYM, ASYM2, ASYM3):
        packing, Q, rmax = ASYM2, 535, 1
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
    v = args.steps * blocks_per_step * geom.W / dt
    line = {"metric": METRIC, "value": v, "unit": "output samples/s",
            "impl": "reference", "n_gpus": D.ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": name, "point": head, "L": len(s), "N": len(k), "W_block": geom.W_block,
                       "step": f"{blocks_per_step} overlap-save blocks (bounded sample of the workload)"},
            "cpu_baseline": {"value": v, "unit": "output samples/s", "cores": 1, "kind": "oracle",
                             "sample": f"{blocks_per_step} blocks per step, NumPy oracle single-threaded"},
            "e2e": {"value": v, "unit": "output samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ our arm
def roofline(rec, head_pt, alg_bytes_per_gpu, traffic=None, traffic_src=None):
    if "fp64_tflops" in rec:
        # the DMMA-core kernel is bound by the FP64 tensor pipe (its own measured peak), the FMA
        # core by the FP64 FMA pipe; adaptive plans: asym2/full launches run DMMA
        mma = bool(rec.get("core_mma")) or head_pt[0] == ADAPT
        peak = MEASURED_DMMA_TFLOPS if mma else MEASURED_FP64_TFLOPS
        return {"bound": "tensor" if mma else "alu", "achieved": rec["fp64_tflops"], "peak": peak, "unit": "TFLOP/s",
                "frac": rec["fp64_tflops"] / peak, "traffic": traffic, "traffic_unit": "bytes/launch",
                "traffic_source": traffic_src, "algorithmic_bytes_per_gpu": alg_bytes_per_gpu,
                "peak_source": DMMA_PEAK_SOURCE if mma else FP64_PEAK_SOURCE,
                "fp64_fma_peak_frac": rec["fp64_tflops"] / MEASURED_FP64_TFLOPS,
                "algorithmic": "FP64 FMAs of the packed core: sum over blocks of M_out * K (2 flop each), per GPU, "
                               "over the max-over-ranks step time"}
    hbm, src = hbm_peak()
    gbs = rec["hbm_gbs_algorithmic"]
    return {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm, "traffic": traffic,
            "peak_source": src, "algorithmic": "8 B read per input sample + 8 B written per output, per GPU"}


def ncu_traffic(kname_prefix, prof_names):
    """dram bytes (read + write) of one launch of the kernel from a committed ncu summary."""
    for prof in prof_names:
        path = os.path.join(ROOT, "profiles", prof)
        if not os.path.exists(path):
            continue
        for recd in json.load(open(path)).get("ncu_full", []):
            if kname_prefix in recd["kernel"]:
                mult = {"Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9, "byte": 1.0}
                rd, wr = recd["dram__bytes_read.sum"].split(), recd["dram__bytes_write.sum"].split()
                return float(rd[0]) * mult[rd[1]] + float(wr[0]) * mult[wr[1]], f"profiles/{prof} (ncu --set full)"
    return None, None


def summarize(name, results, head, full_pt, meta, scaling, D):
    h = results[head]
    full = results.get(full_pt)
    pt = WORKLOADS[name][1][head]
    alg = None if name == "cfg4" else 8 * (2 * meta["L"] + meta["N"] - 1) // D.ws
    traffic, tsrc = None, None
    if name == "cfg2" and head == "asym2_10b":
        traffic, tsrc = ncu_traffic(f"pc_tiled_kernel<2, {h['tile']}, {h['core_mma']}",   # (+ ", 0>" since r02b)
                                    ["r02b_ncu_cfg2_asym2.json", "r02_ncu_cfg2_asym2.json", "r01_ncu_cfg2_asym2_dmma.json"])
    roof = roofline(h, pt, alg, traffic, tsrc)
    if h.get("core") == "fft":
        roof["kernel"] = "pc_fft_conv_kernel"
    elif pt[0] == ADAPT:
        roof["kernel"] = "pc_tiled_kernel x3 (one launch per packing) + pc_block_stats/pc_adapt_decide/pc_adapt_lists"
    elif h.get("exec") == 2:
        roof["kernel"] = f"pc_tiled_kernel<{pt[0]}, {h.get('tile')}, {h.get('core_mma')}>"
    else:
        roof["kernel"] = "pc_fused_kernel (one CTA per block)"
    out = {"workload": name, "point": head, "value": h["value"], "unit": "output samples/s",
           "ms_per_step": h["ms_per_step"], "scaling": scaling, "roofline": roof,
           "packed_vs_full": (h["value"] / full["value"]) if full else None, "points": results,
           "config": {k: v for k, v in meta.items() if k != "per_buf"}}
    if name == "cfg3" and "full_fft" in results:
        out["packed_vs_full_fair_circular"] = h["value"] / results["full_fft"]["value"]
    return out


def run_ours(args, D):
    import torch
    dev = torch.device("cuda", D.local)
    name = args.workload
    W_block, points, head, full_pt = WORKLOADS[name]
    sel = [p for p in (args.points.split(",") if args.points else points) if p in points]
    if head not in sel:                                # diagnostics subset: first selected point leads
        head = sel[0]
    x_k = None
    if name == "cfg4":
        res, clocks, meta = measure_cfg4(sel, head, args, D, dev, args.signals or 1024, clocks=True)
        scaling = "strong"
    else:
        weak = name in ("cfg1", "cfg2")                # cfg2 headline: N x 2^22 samples (fixed work per GPU)
        scaling = "weak" if weak else "strong"
        L_g = (args.L or BASE_L[name]) * (D.ws if weak else 1)
        res, clocks, meta, x_k = measure_split(name, sel, head, args, D, dev, L_g, clocks=True, N_override=args.N)
    main_rec = summarize(name, res, head, full_pt, meta, scaling, D)
    subs = {}
    if name == "cfg2" and not args.no_sub and not args.points:
        for sub in ("cfg3", "cfg5"):
            r_, _, m_, _ = measure_split(sub, SUB_POINTS[sub], WORKLOADS[sub][2], args, D, dev, BASE_L[sub])
            subs[sub] = summarize(sub, r_, WORKLOADS[sub][2], WORKLOADS[sub][3], m_, "strong", D)
        r_, _, m_ = measure_cfg4(SUB_POINTS["cfg4"], "asym2_8b", args, D, dev, args.cfg4_signals * D.ws)
        subs["cfg4"] = summarize("cfg4", r_, "asym2_8b", "full", m_, "weak", D)
        subs["cfg4"]["config"]["note"] = (f"bounded database: {args.cfg4_signals} of BASELINE.json's 1024 signals per "
                                          f"rank (the full 1024 x 2^20 runs with --workload cfg4)")
    if D.rank != 0:
        return
    h = res[head]
    launches = {ADAPT: 6}.get(points[head][0], 4 if name == "cfg4" else 1)
    line = {
        "metric": METRIC,
        "value": h["value"], "unit": "output samples/s", "n_gpus": D.ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": h["ms_per_step"], "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": name, "L": meta["L"], "N": meta["N"], "W_block": meta["W_block"], "point": head,
                   "l2": (f"inputs larger than L2: {meta.get('n_buf', 1)} rotating input/output buffer pairs per rank "
                          f"({meta.get('n_buf', 1) * meta.get('per_buf', 0) >> 20} MiB)" if name != "cfg4" else
                          "inputs larger than L2 (the rank's database shard)"),
                   "parallelism": (f"{D.ws} rank(s), one signal split by overlap-save block range "
                                   f"(conv_shard_range + conv_execute_blocks, N'+1-sample halo)" if name != "cfg4" else
                                   f"{D.ws} rank(s), database sharded by signal + NCCL gather of the winners"),
                   "process_group": D.backend, "early_fill": 1},
        "gpu_launches": args.steps * launches,
        "roofline": main_rec["roofline"],
        "e2e": h.get("e2e"),
        "packed_vs_full": main_rec["packed_vs_full"],
        "full_precision": res.get(full_pt),
        "points": res,
        "clocks": clocks,
        "sub_records": subs,
        # the paper's own numbers: context only, another machine and workload
        "paper_context": {"hardware": "Intel Core i5 540M 2.5 GHz, single-threaded, Intel IPP 7.0 ippsConv_64f "
                                      "(P:153, P:164)",
                          "packed_vs_full": {"synthetic_IV_A_sym": "+52%..+158% (Table 2, P:176-181)",
                                             "music_matching_xcorr_sym": "+112.5% (Table 3, P:195-199)",
                                             "mpeg7_xcorr_sym": "+174% (Table 4, P:207-212)"},
                          "best_msamples_per_s": 15.57},
    }
    if "packed_vs_full_fair_circular" in main_rec:
        line["packed_vs_full_fair_circular"] = main_rec["packed_vs_full_fair_circular"]
    if D.ws == 1 and not args.no_cpu_baseline and x_k is not None:
        x, k = x_k
        line["cpu_baseline"] = cpu_baseline(x, k, W_block, points[head])
        line["cpu_baseline_all_cores"] = cpu_baseline_all_cores(x, k, W_block, points[head])
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    D = Dist(args)
    try:
        if args.impl == "reference":
            run_reference(args, D)
        else:
            run_ours(args, D)
        D.barrier()
    finally:
        D.close()


if __name__ == "__main__":
    main()
