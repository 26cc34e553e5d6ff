"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bar (task rule ③): companding factors, packed words, packed convolution
outputs (dyadic eps: exact arithmetic), unpacked integers and dequantized outputs are
BIT-EXACT; full-precision outputs are within 1e-12 normalized L-inf (north_star,
reading C16).  Sizes span several tiles and ragged tails; full BASELINE sizes are
checked on sampled blocks the oracle computes one by one.
"""
import math

import numpy as np
import pytest

import oracle as O
from paper_1201_3018_b200 import workloads as WL

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1201_3018_b200 import binding as pcb
    DEV = torch.device("cuda:0")

PK = {O.FULL: 0, O.SYM: 1, O.ASYM2: 2, O.ASYM3: 3}
EPS = {O.EPS_PAPER: 0, O.EPS_RADIX: 1, O.EPS_POW2: 2}


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


def gpu_run(s, k, W_block, packing, Q, mode=O.CONV, eps_rule=O.EPS_POW2, rmax_rule=O.RMAX_PAPER, debug=True,
            tile=0, npart=0, exec_=0, core=0):
    opts = pcb.opts_default(eps_rule=EPS[eps_rule], rmax_rule=rmax_rule, bound_policy=pcb.BOUND_WARN, exec=exec_)
    opts.core_tile = tile
    opts.core_variant = core    # direct core: 0 auto (FP64 tensor cores, T = 16), 1 FP64 FMA, 2 DMMA
    opts.parts_per_job = npart
    with pcb.Plan(len(s), len(k), W_block, mode, PK[packing], Q, opts=opts) as p:
        p.set_kernel(dev(k))
        info = p.info()
        s_d = dev(s)
        r = torch.full((info["L_out"],), float("nan"), dtype=torch.float64, device=DEV)
        out = {"info": info}
        if debug:
            P = info["P"]
            packed = torch.zeros((P, info["packed_stride"]), dtype=torch.float64, device=DEV)
            rbar = torch.zeros((P, info["rbar_stride"]), dtype=torch.float64, device=DEV)
            rint = torch.zeros((P, info["rint_stride"]), dtype=torch.int64, device=DEV)
            cs = torch.zeros(P, dtype=torch.float64, device=DEV)
            p.execute_debug(s_d, r, packed, rbar, rint, cs)
            torch.cuda.synchronize()
            out.update(packed=packed.cpu().numpy(), rbar=rbar.cpu().numpy(), rint=rint.cpu().numpy(),
                       cs=cs.cpu().numpy(), r_dbg=r.cpu().numpy())
            r.fill_(float("nan"))
        p.execute(s_d, r)
        torch.cuda.synchronize()
        out["r"] = r.cpu().numpy()
    return out


def check_blocks(g, ref, packing):
    """Per-step bit-exact comparison against the oracle's per-block record."""
    geom = ref.geom
    for br in ref.blocks:
        w = br.w
        o0, n_out = geom.kept(w)
        if packing != O.FULL:
            assert g["cs"][w] == br.c_s, ("c_s", w)
            assert np.array_equal(g["packed"][w, :br.packed.shape[0]], br.packed), ("packed words", w)
            assert np.array_equal(g["rbar"][w, :br.rbar.shape[0]], br.rbar), ("packed conv outputs", w)
            assert np.array_equal(g["rint"][w, :n_out], br.r_int.astype(np.int64)), ("unpacked integers", w)
            assert np.array_equal(g["rint"][w, :n_out], br.r_exact), ("exact integer conv", w)


SMALL_CASES = [  # (L, N, W_block, Q): several tiles, ragged tails, P = 1, N = 1, N > L
    (1000, 9, 40, 7), (777, 10, 34, 7), (5, 1, 4, 3), (4097, 64, 1024, 127), (20000, 513, 4096, 31),
    (3, 2, 10, 5), (5, 9, 30, 3), (70000, 65, 1024, 60), (12345, 255, 2048, 15),
]


@pytest.mark.parametrize("exec_,core", [(0, 0), (2, 2), (2, 1), (1, 0)])   # auto, tiled DMMA / FMA, per-block
@pytest.mark.parametrize("packing", [O.SYM, O.ASYM2, O.ASYM3])
@pytest.mark.parametrize("case", SMALL_CASES)
def test_packed_bit_exact_pow2(packing, case, exec_, core):
    L, N, W_block, Q = case
    rng = np.random.default_rng(L * 7 + N)
    s, k = rng.laplace(0, 0.3, L), rng.uniform(-1, 1, N)
    Np = N | 1
    Q = min(Q, O.max_q_under_bound(None, Np, packing, O.EPS_POW2, O.RMAX_PAPER))   # Eq. (3) within bound
    ref = O.conv_pipeline(s, k, W_block, packing, Q, keep_blocks=True)
    assert ref.kernel.bound_ok and ref.mismatches == 0
    g = gpu_run(s, k, W_block, packing, Q, exec_=exec_, core=core)
    assert g["info"]["c_k"] == ref.kernel.c_k and g["info"]["R_max"] == ref.kernel.R
    assert g["info"]["eps_inv"] == ref.kernel.eps.eps_inv
    check_blocks(g, ref, packing)
    assert np.array_equal(g["r_dbg"], ref.out)
    assert np.array_equal(g["r"], ref.out)


@pytest.mark.parametrize("tile,core", [(12, 1), (14, 1), (16, 1), (16, 2)])
@pytest.mark.parametrize("packing", [O.FULL, O.SYM, O.ASYM2, O.ASYM3])
@pytest.mark.parametrize("case", [(20000, 513, 4096, 31), (4097, 64, 1024, 60), (9000, 100, 512, 15)])
def test_every_core_tile(tile, core, packing, case):
    """The tiled kernel's core: the FP64 FMA loop at T = 12/14/16 and the FP64 tensor-core
    (DMMA) Toeplitz core at T = 16; force each one."""
    L, N, W_block, Q = case
    rng = np.random.default_rng(N + tile)
    s, k = rng.laplace(0, 0.3, L), rng.uniform(-1, 1, N)
    if packing == O.FULL:
        g = gpu_run(s, k, W_block, O.FULL, 0, debug=False, tile=tile, core=core)
        want = O.full_precision(s, k)
        assert np.max(np.abs(g["r"] - want)) / np.max(np.abs(want)) < 1e-12
        return
    Q = min(Q, O.max_q_under_bound(None, N | 1, packing, O.EPS_POW2, O.RMAX_PAPER))
    ref = O.conv_pipeline(s, k, W_block, packing, Q)
    g = gpu_run(s, k, W_block, packing, Q, debug=False, tile=tile, core=core)
    assert np.array_equal(g["r"], ref.out)


@pytest.mark.parametrize("core", [2, 1])
@pytest.mark.parametrize("npart", [1, 2, 4])
@pytest.mark.parametrize("packing", [O.FULL, O.SYM, O.ASYM2, O.ASYM3])
@pytest.mark.parametrize("mode", [O.CONV, O.XCORR])
def test_every_parts_per_job(npart, packing, mode, core):
    """The tiled kernel splits a job into npart warp parts (G = 32 npart groups), each claimed
    by a consumer warp of one SM sub-partition; force each split (ring depth, sentinel count
    16/npart and the per-warp symmetric B hand-over all change with it)."""
    L, N, W_block, Q = 150_000, 201, 2048, 31
    rng = np.random.default_rng(npart * 10 + packing)
    s, k = np.clip(rng.laplace(0, 0.3, L), -1, 1), rng.uniform(-1, 1, N)
    if packing == O.FULL:
        g = gpu_run(s, k, W_block, O.FULL, 0, mode=mode, debug=False, npart=npart, core=core)
        want = O.full_precision(s, k, mode=mode)
        assert np.max(np.abs(g["r"] - want)) / np.max(np.abs(want)) < 1e-12
        return
    Q = min(Q, O.max_q_under_bound(None, N | 1, packing, O.EPS_POW2, O.RMAX_PAPER))
    ref = O.conv_pipeline(s, k, W_block, packing, Q, mode=mode)
    g = gpu_run(s, k, W_block, packing, Q, mode=mode, debug=False, npart=npart, core=core)
    assert np.array_equal(g["r"], ref.out)


def test_graph_replay_bit_exact():
    """Job queues are reset by the last CTA of every launch, so a captured CUDA graph of
    several executions replays with identical results (no host-side counter state)."""
    L, N, W_block, Q = 300_000, 513, 4096, 511
    s, k = WL.cfg2(seed=3, L=L, N=N)
    ref = O.conv_pipeline(s, k, W_block, O.ASYM2, Q, rmax_rule=O.RMAX_L1).out
    with pcb.Plan(L, N, W_block, pcb.MODE_CONV, pcb.PACK_ASYM2, Q, rmax_rule=pcb.RMAX_L1) as p:
        p.set_kernel(dev(k))
        S = dev(s)
        R = [torch.full((L + N - 1,), float("nan"), dtype=torch.float64, device=DEV) for _ in range(3)]
        p.execute(S, R[0])
        torch.cuda.synchronize()
        gs = torch.cuda.Stream(DEV)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(gs):
            with torch.cuda.graph(graph, stream=gs):
                for r in R:
                    p.execute(S, r)
        for _ in range(3):
            for r in R:
                r.fill_(float("nan"))
            graph.replay()
            torch.cuda.synchronize()
            for r in R:
                assert np.array_equal(r.cpu().numpy(), ref)


@pytest.mark.parametrize("packing", [O.SYM, O.ASYM2, O.ASYM3])
@pytest.mark.parametrize("eps_rule", [O.EPS_PAPER, O.EPS_RADIX])
def test_packed_integers_exact_nondyadic_eps(packing, eps_rule):
    """Non-dyadic eps: packed words are deterministic (bit-exact); the core's FMA order may
    change the last bits of r_bar, but the unpacked integers are exact (within bound)."""
    L, N, W_block, Q = 20000, 65, 1024, 5
    rng = np.random.default_rng(11)
    s, k = rng.laplace(0, 0.3, L), rng.uniform(-1, 1, N)
    ref = O.conv_pipeline(s, k, W_block, packing, Q, eps_rule=eps_rule, keep_blocks=True)
    assert ref.kernel.bound_ok and ref.mismatches == 0
    g = gpu_run(s, k, W_block, packing, Q, eps_rule=eps_rule)
    for br in ref.blocks:
        o0, n_out = ref.geom.kept(br.w)
        assert np.array_equal(g["packed"][br.w, :br.packed.shape[0]], br.packed)
        assert np.array_equal(g["rint"][br.w, :n_out], br.r_exact)
    assert np.array_equal(g["r"], ref.out)


@pytest.mark.parametrize("case", SMALL_CASES)
def test_full_precision_within_1e12(case):
    L, N, W_block, _ = case
    rng = np.random.default_rng(L + 3 * N)
    s, k = rng.normal(size=L), rng.normal(size=N)
    want = O.full_precision(s, k)
    g = gpu_run(s, k, W_block, O.FULL, 0, debug=False)
    err = np.max(np.abs(g["r"] - want)) / np.max(np.abs(want))
    assert err < 1e-12, err


@pytest.mark.parametrize("packing", [O.FULL, O.SYM, O.ASYM2])
def test_xcorr_mode(packing):
    rng = np.random.default_rng(5)
    s, q = rng.laplace(0, 0.3, 9000), rng.uniform(-1, 1, 100)
    Q = {O.FULL: 0, O.SYM: 31, O.ASYM2: 63}[packing]          # within Table 1 / dyadic bounds
    ref = O.conv_pipeline(s, q, 512, packing, Q, mode=O.XCORR, keep_blocks=True)
    g = gpu_run(s, q, 512, packing, Q, mode=O.XCORR, debug=packing != O.FULL)
    assert g["r"].shape == (9000 - 100 + 1,)
    if packing == O.FULL:
        want = O.full_precision(s, q, O.XCORR)
        assert np.max(np.abs(g["r"] - want)) / np.max(np.abs(want)) < 1e-12
    else:
        assert ref.mismatches == 0
        check_blocks(g, ref, packing)
        assert np.array_equal(g["r"], ref.out)


def test_edge_cases_zero_delta_saturating():
    rng = np.random.default_rng(8)
    s = rng.uniform(-1, 1, 3000)
    s[500:1500] = 0.0                                            # all-zero blocks: c_s = 1
    for packing in (O.SYM, O.ASYM2, O.ASYM3):
        for k in ([1.0], [0.0, 0.0, 0.0], rng.uniform(-1, 1, 9)):   # delta, zero kernel, random
            ref = O.conv_pipeline(s, k, 40, packing, 15, keep_blocks=True)
            g = gpu_run(s, k, 40, packing, 15)
            check_blocks(g, ref, packing)
            assert np.array_equal(g["r"], ref.out)
    # square wave matched to the kernel signs: outputs reach +R_max (L1 rule, reading C3)
    k = rng.uniform(-1, 1, 9)
    k_int, _, _ = O.compand(k, 5)
    sq = np.tile(np.sign(k_int[::-1]) + (k_int[::-1] == 0), 40)
    ref = O.conv_pipeline(sq, k, 40, O.SYM, 5, rmax_rule=O.RMAX_L1, keep_blocks=True)
    assert max(int(np.max(b.r_exact)) for b in ref.blocks) == ref.kernel.R
    g = gpu_run(sq, k, 40, O.SYM, 5, rmax_rule=O.RMAX_L1)
    check_blocks(g, ref, O.SYM)
    assert np.array_equal(g["r"], ref.out)


def test_bound_policy_strict():
    k = np.ones(513)
    with pcb.Plan(10000, 513, 4096, pcb.MODE_CONV, pcb.PACK_SYM, 127) as p:   # 513*127^2 > 131071
        with pytest.raises(pcb.PcError) as ei:
            p.set_kernel(dev(k))
        assert ei.value.code == pcb.PC_E_BOUND


@pytest.mark.parametrize("mode", [O.CONV, O.XCORR])
def test_execute_blocks_sharding_bit_identical(mode):
    """Block-range sharding: each 'rank' takes its shard from conv_shard_range,
    holds only its input slice plus the N'+1 halo, and runs conv_execute_blocks; the union of
    the shards' outputs is bit-identical to the single run, for G = 1, 2, 3, 4, 8."""
    rng = np.random.default_rng(2)
    L, N, W_block, Q = 200000, 64, 1024, 255
    s, k = rng.laplace(0, 0.2, L), rng.uniform(-1, 1, N)
    ref = O.conv_pipeline(s, k, W_block, O.ASYM2, Q, mode=mode)
    with pcb.Plan(L, N, W_block, mode, pcb.PACK_ASYM2, Q) as p:
        p.set_kernel(dev(k))
        info = p.info()
        for G in (1, 2, 3, 4, 8):
            out = np.full(info["L_out"], np.nan)
            covered = 0
            for rank in range(G):
                sh = pcb.shard_range(L, N, W_block, mode, rank, G)
                in0, in1, o0, o1 = sh["in_begin"], sh["in_end"], sh["out_begin"], sh["out_end"]
                s_slice = dev(s[in0:in1])
                r_slice = torch.full((max(1, o1 - o0),), float("nan"), dtype=torch.float64, device=DEV)
                p.execute_blocks(s_slice, in0, r_slice, o0, sh["block_begin"], sh["block_end"])
                torch.cuda.synchronize()
                assert np.isnan(out[o0:o1]).all()          # disjoint output ranges
                out[o0:o1] = r_slice[:o1 - o0].cpu().numpy()
                covered += o1 - o0
            assert covered == info["L_out"]
            assert np.array_equal(out, ref.out), G


def test_execute_batch_and_host_and_misaligned():
    rng = np.random.default_rng(3)
    L, N, W_block, Q = 50000, 100, 1024, 127
    k = rng.uniform(-1, 1, N)
    S = rng.laplace(0, 0.2, (3, L))
    refs = [O.conv_pipeline(S[i], k, W_block, O.ASYM2, Q).out for i in range(3)]
    with pcb.Plan(L, N, W_block, pcb.MODE_CONV, pcb.PACK_ASYM2, Q) as p:
        p.set_kernel(dev(k))
        Lo = L + N - 1
        R = torch.full((3, Lo + 5), float("nan"), dtype=torch.float64, device=DEV)
        Sd = torch.zeros((3, L + 3), dtype=torch.float64, device=DEV)
        Sd[:, :L] = dev(S)
        p.execute_batch(Sd, 3, L + 3, R, Lo + 5)
        torch.cuda.synchronize()
        for i in range(3):
            assert np.array_equal(R[i, :Lo].cpu().numpy(), refs[i])
        # host buffers (pinned) through conv_execute_host
        sh = torch.from_numpy(S[1].copy()).pin_memory()
        rh = torch.empty(Lo, dtype=torch.float64).pin_memory()
        p.execute_host(sh, rh)
        assert np.array_equal(rh.numpy(), refs[1])
        # misaligned input pointer (8-byte offset): plain-load staging path, same bits
        buf = torch.zeros(L + 1, dtype=torch.float64, device=DEV)
        buf[1:] = dev(S[2])
        r = torch.empty(Lo, dtype=torch.float64, device=DEV)
        p.execute(buf[1:], r)
        torch.cuda.synchronize()
        assert np.array_equal(r.cpu().numpy(), refs[2])


@pytest.mark.parametrize("floor", [20.0, 30.0, 40.0, 50.0, 60.0, math.inf])
def test_adaptive_decisions_and_output(floor):
    s, k = WL.cfg5(seed=1, L=1 << 17, N=1024)
    W_block = 4096
    y_ref, dec_ref, qmode = O.adaptive_pipeline(s, k, W_block, floor)
    with pcb.Plan(len(s), len(k), W_block, pcb.MODE_CONV, pcb.PACK_ADAPTIVE, 0, rmax_rule=pcb.RMAX_L1) as p:
        p.set_kernel(dev(k))
        info = p.info()
        assert info["q_mode"][1] == qmode[O.SYM] and info["q_mode"][2] == qmode[O.ASYM2]
        s_d = dev(s)
        dec = p.adapt_block(s_d, floor)
        assert [(d[0], d[1]) for d in dec] == [(PK[m], q) for m, q, _ in dec_ref]
        assert [d[2] for d in dec] == [x[2] for x in dec_ref]
        r = torch.empty(info["L_out"], dtype=torch.float64, device=DEV)
        p.execute(s_d, r)
        torch.cuda.synchronize()
        got = r.cpu().numpy()
    # packed blocks bit-exact; full-precision blocks (SNR = inf) within 1e-12 (C16)
    geom = O.Geometry(len(s), len(k), W_block)
    for w, (m, q, _) in enumerate(dec_ref):
        g0 = geom.block_start(w)
        o0, n_out = geom.kept(w)
        lo, hi = g0 + o0, min(g0 + o0 + n_out, geom.L_out)
        if m == O.FULL:
            scale = max(np.max(np.abs(y_ref[lo:hi])), 1e-300)
            assert np.max(np.abs(got[lo:hi] - y_ref[lo:hi])) / scale < 1e-12, w
        else:
            assert np.array_equal(got[lo:hi], y_ref[lo:hi]), w


@pytest.mark.parametrize("exec_", [0, 1])    # auto (tiled kernel, fused score epilogue), per-block + lag scan
def test_xcorr_max_scores(exec_):
    """conv_xcorr_max: per-signal max over valid lags and its lowest argmax (C17).  The tiled
    kernel fuses the score into its epilogue (warp partials + a per-signal reduction, no lag
    buffer); the per-block kernel stores the lags and scans them.  Both equal the oracle."""
    rng = np.random.default_rng(4)
    n_sig, L, N = 6, 1 << 14, 256
    db = np.stack([WL.cfg4_signal(i, L) for i in range(n_sig)])
    q = db[3, 5000:5000 + N] + rng.normal(0, 0.01, N)
    for packing, Q in ((O.FULL, 0), (O.SYM, 7), (O.ASYM2, 127)):
        with pcb.Plan(L, N, 2048, pcb.MODE_XCORR, PK[packing], Q, rmax_rule=pcb.RMAX_L1, exec=exec_) as p:
            p.set_kernel(dev(q))
            sc = torch.empty(n_sig, dtype=torch.float64, device=DEV)
            lag = torch.empty(n_sig, dtype=torch.int64, device=DEV)
            p.xcorr_max(dev(db), n_sig, L, sc, lag)
            torch.cuda.synchronize()
            sc, lag = sc.cpu().numpy(), lag.cpu().numpy()
        for i in range(n_sig):
            if packing == O.FULL:
                c = O.full_precision(db[i], q, O.XCORR)
                best, j = O.xcorr_score(c)
                assert abs(sc[i] - best) <= 1e-12 * np.max(np.abs(c))
                assert c[lag[i]] >= best - 1e-12 * np.max(np.abs(c))
            else:
                c = O.conv_pipeline(db[i], q, 2048, packing, Q, mode=O.XCORR, rmax_rule=O.RMAX_L1).out
                assert (sc[i], lag[i]) == O.xcorr_score(c)
        assert int(np.argmax(sc)) == 3 and lag[3] == 5000


# --------------------------------------------------------------------- full BASELINE sizes
def _sampled_full_size(s, k, W_block, packing, Q, rmax_rule, min_snr):
    geom = O.Geometry(len(s), len(k), W_block)
    blocks = sorted({0, 1, 2, geom.P // 3, geom.P // 2, geom.P - 2, geom.P - 1})
    ref = O.conv_pipeline(s, k, W_block, packing, Q, rmax_rule=rmax_rule, blocks=blocks)
    g = gpu_run(s, k, W_block, packing, Q, rmax_rule=rmax_rule, debug=False)
    sel = ~np.isnan(ref.out)
    assert np.array_equal(g["r"][sel], ref.out[sel])
    assert ref.mismatches == 0
    assert not np.any(np.isnan(g["r"]))
    return g


@pytest.mark.parametrize("packing,Q,rmax,min_snr", [(O.ASYM2, 511, O.RMAX_L1, 40.0), (O.SYM, 127, O.RMAX_L1, 30.0),
                                                    (O.ASYM3, 127, O.RMAX_L1, 30.0), (O.ASYM2, 31, O.RMAX_PAPER, 20.0)])
def test_cfg2_full_size_sampled(packing, Q, rmax, min_snr):
    s, k = WL.cfg2(seed=0)
    g = _sampled_full_size(s, k, 4096, packing, Q, rmax, min_snr)
    full = O.full_precision(s[:1 << 18], k)
    snr = O.measured_snr_db(full[:(1 << 18)], g["r"][:1 << 18])
    assert snr >= min_snr, snr


@pytest.mark.parametrize("packing,Q", [(O.ASYM2, 511), (O.SYM, 127), (O.ASYM3, 127)])
@pytest.mark.parametrize("opt", ["producer_sms", "pack_alu"])
def test_cfg2_full_size_producer_variants(packing, Q, opt):
    """The persistent kernel's alternative producers at full cfg2 size: the producer-SM mode
    (conv_opts.prepack = -16: CTAs 0..15 pack jobs 528.. into stage images in HBM and flag them,
    the others bulk-copy them after their own pipeline fill) and integer/FP32 companding and
    packing (pack_alu = 1, pc_intfp.cuh) -- bit-exact with the oracle on sampled blocks (blocks
    past the fills included) and bit-identical with the default fused path everywhere."""
    s, k = WL.cfg2(seed=0)
    geom = O.Geometry(len(s), len(k), 4096)
    blocks = sorted({0, 1, geom.P // 2, geom.P - 2, geom.P - 1})
    ref = O.conv_pipeline(s, k, 4096, packing, Q, rmax_rule=O.RMAX_L1, blocks=blocks)
    outs = []
    for variant in (0, 1):
        opts = pcb.opts_default(rmax_rule=pcb.RMAX_L1)
        if variant:
            if opt == "producer_sms":
                opts.prepack = -16
            else:
                opts.pack_alu = 1
        with pcb.Plan(len(s), len(k), 4096, pcb.MODE_CONV, PK[packing], Q, opts=opts) as p:
            p.set_kernel(dev(k))
            r = torch.full((p.info()["L_out"],), float("nan"), dtype=torch.float64, device=DEV)
            for _ in range(3):                   # repeated launches: epochs / queues / flags reused
                p.execute(dev(s), r)
            torch.cuda.synchronize()
            outs.append(r.cpu().numpy())
    sel = ~np.isnan(ref.out)
    assert np.array_equal(outs[1][sel], ref.out[sel])
    assert not np.any(np.isnan(outs[1]))
    assert np.array_equal(outs[0], outs[1])


def test_cfg2_full_precision_full_size():
    s, k = WL.cfg2(seed=0)
    g = gpu_run(s, k, 4096, O.FULL, 0, debug=False)
    want = O.full_precision(s, k)
    assert np.max(np.abs(g["r"] - want)) / np.max(np.abs(want)) < 1e-12


def test_cfg1_full_size_all_packings():
    s, k = WL.cfg1(seed=0)
    for packing, Q in ((O.ASYM2, 127), (O.ASYM2, 255), (O.SYM, 44), (O.ASYM3, 15)):
        ref = O.conv_pipeline(s, k, 1024, packing, Q, keep_blocks=True)
        assert ref.kernel.bound_ok and ref.mismatches == 0
        g = gpu_run(s, k, 1024, packing, Q)
        check_blocks(g, ref, packing)
        assert np.array_equal(g["r"], ref.out)


# --------------------------------------------------------------------- large kernels: tap chunks, tiles
@pytest.mark.parametrize("core", [2, 1])
@pytest.mark.parametrize("packing", [O.FULL, O.SYM, O.ASYM2, O.ASYM3])
@pytest.mark.parametrize("case", [(70000, 4096, 16384), (40000, 1024, 16384), (100000, 8192, 32768)])
def test_large_kernels_tap_chunks_and_tiles(packing, case, core):
    """cfg3/cfg4-shaped geometries: taps processed in chunks, blocks split into several
    output tiles (the symmetric tile boundary uses the extra-word path)."""
    L, N, W_block = case
    rng = np.random.default_rng(N)
    s, k = rng.laplace(0, 0.3, L), rng.normal(0, 1 / np.sqrt(N), N)
    if packing == O.FULL:
        g = gpu_run(s, k, W_block, O.FULL, 0, debug=False, core=core)
        want = O.full_precision(s, k)
        assert np.max(np.abs(g["r"] - want)) / np.max(np.abs(want)) < 1e-12
        return
    Q = 3 if packing != O.ASYM2 else 127
    ref = O.conv_pipeline(s, k, W_block, packing, Q, rmax_rule=O.RMAX_L1)
    assert ref.kernel.bound_ok and ref.mismatches == 0
    g = gpu_run(s, k, W_block, packing, Q, rmax_rule=O.RMAX_L1, debug=False, core=core)
    assert np.array_equal(g["r"], ref.out)


def test_cfg4_shaped_xcorr_large_query():
    rng = np.random.default_rng(7)
    L, N = 1 << 17, 8192
    x = WL.cfg4_signal(3, L)
    q = x[40000:40000 + N] + rng.normal(0, 0.01, N)
    for packing, Q in ((O.ASYM2, 127), (O.SYM, 3)):
        ref = O.conv_pipeline(x, q, 32768, packing, Q, mode=O.XCORR, rmax_rule=O.RMAX_L1)
        assert ref.kernel.bound_ok and ref.mismatches == 0
        g = gpu_run(x, q, 32768, packing, Q, mode=O.XCORR, rmax_rule=O.RMAX_L1, debug=False)
        assert np.array_equal(g["r"], ref.out)
        assert int(np.argmax(g["r"])) == 40000


# --------------------------------------------------------------------- full BASELINE sizes (sampled)
def test_cfg3_full_size_direct_sampled():
    """Config 3 at full size (L = 2^24, N = 4096, W_block = 16384) on the direct core: asym2
    9-bit (L1, dyadic) bit-exact on sampled blocks; full precision within 1e-12 on a window."""
    s, k = WL.cfg3(seed=0)
    _sampled_full_size(s, k, 16384, O.ASYM2, 255, O.RMAX_L1, 40.0)
    g = gpu_run(s, k, 16384, O.FULL, 0, debug=False)
    lo, hi = 5_000_000, 5_000_000 + 20000
    want = np.convolve(s[lo - 4095:hi], k)[4095:4095 + (hi - lo)]
    got = g["r"][lo:hi]
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 1e-12


def test_cfg4_full_size_signals_scores():
    """Config 4 shape: 2^20-sample database signals, N = 8192 query, W_block = 32768; packed
    scores/lags bit-exact against the oracle on 3 signals; the query's source signal wins."""
    n_sig, L, N = 3, 1 << 20, 8192
    q, i0, off = WL.cfg4_query(seed=0, n_signals=n_sig, L=L, N=N)
    db = np.stack([WL.cfg4_signal(i, L) for i in range(n_sig)])
    with pcb.Plan(L, N, 32768, pcb.MODE_XCORR, pcb.PACK_ASYM2, 127, rmax_rule=pcb.RMAX_L1) as p:
        p.set_kernel(dev(q))
        sc = torch.empty(n_sig, dtype=torch.float64, device=DEV)
        lag = torch.empty(n_sig, dtype=torch.int64, device=DEV)
        p.xcorr_max(dev(db), n_sig, L, sc, lag)
        torch.cuda.synchronize()
        sc, lag = sc.cpu().numpy(), lag.cpu().numpy()
    for i in range(n_sig):
        c = O.conv_pipeline(db[i], q, 32768, O.ASYM2, 127, mode=O.XCORR, rmax_rule=O.RMAX_L1).out
        assert (sc[i], lag[i]) == O.xcorr_score(c)
    assert int(np.argmax(sc)) == i0 and lag[i0] == off


def test_cfg5_full_size_adaptive_sampled():
    """Config 5 at full size (L = 2^26, N = 1024, W_block = 4096), floor 40 dB: every block's
    decision equals the oracle's; outputs bit-exact (packed) / 1e-12 (full) on sampled blocks."""
    s, k = WL.cfg5(seed=0)
    W_block, floor = 4096, 40.0
    dec_ref, qmode = O.adapt_decisions(s, k, W_block, floor)
    geom = O.Geometry(len(s), len(k), W_block)
    with pcb.Plan(len(s), len(k), W_block, pcb.MODE_CONV, pcb.PACK_ADAPTIVE, 0, rmax_rule=pcb.RMAX_L1) as p:
        p.set_kernel(dev(k))
        s_d = dev(s)
        dec = p.adapt_block(s_d, floor)
        assert [(d[0], d[1]) for d in dec] == [(PK[m], q) for m, q, _ in dec_ref]
        r = torch.empty(geom.L_out, dtype=torch.float64, device=DEV)
        p.execute(s_d, r)
        torch.cuda.synchronize()
        got = r.cpu().numpy()
    states = {m: O.prepare_kernel(k, geom, m, qmode[m], None, O.CONV, O.EPS_POW2, O.RMAX_L1) for m in qmode}
    states[O.FULL] = O.prepare_kernel(k, geom, O.FULL, 0)
    for w in sorted({0, 1, geom.P // 2, geom.P - 1}):
        m, Q, _ = dec_ref[w]
        br = O.process_block(s, w, geom, states[m], Q)
        o0, n = geom.kept(w)
        lo = geom.block_start(w) + o0
        n = min(n, geom.L_out - lo)
        if m == O.FULL:
            assert np.max(np.abs(got[lo:lo + n] - br.out[:n])) <= 1e-12 * np.max(np.abs(br.out[:n]))
        else:
            assert np.array_equal(got[lo:lo + n], br.out[:n])


# --------------------------------------------------------------------- FFT core (config 3)
def fft_run(s, k, W_block, packing, Q, mode=O.CONV, rmax_rule=O.RMAX_L1, policy=None):
    opts = pcb.opts_default(core=pcb.CORE_FFT, rmax_rule=rmax_rule,
                            bound_policy=pcb.BOUND_WARN if policy is None else policy)
    with pcb.Plan(len(s), len(k), W_block, mode, PK[packing], Q, opts=opts) as p:
        p.set_kernel(dev(k))
        info = p.info()
        r = torch.full((info["L_out"],), float("nan"), dtype=torch.float64, device=DEV)
        p.execute(dev(s), r)
        torch.cuda.synchronize()
        res, rc = p.residual()
        return r.cpu().numpy(), res, rc, info


@pytest.mark.parametrize("case", [(1 << 18, 4096, 16384), (50000, 1000, 4096), (30000, 63, 1024), (9000, 512, 2048)])
def test_fft_full_precision(case):
    L, N, W_block = case
    rng = np.random.default_rng(N)
    s, k = rng.laplace(0, 0.2, L), rng.normal(0, 1 / np.sqrt(N), N)
    got, _, _, info = fft_run(s, k, W_block, O.FULL, 0)
    want = O.full_precision(s, k)
    assert info["fft_n"] > 0
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 1e-12


@pytest.mark.parametrize("mode", [O.CONV, O.XCORR])
@pytest.mark.parametrize("case", [(1 << 18, 4096, 16384), (100_000, 1000, 8192), (40_000, 3000, 16384),
                                  (20_000, 4096, 16384)])
def test_fft32k_configured_full_precision(case, mode):
    """cfg3's configured full-precision core: the block's linear convolution through a
    32768-point real transform (conv_opts.fft_n = 16384), computed by 2-CTA clusters
    (parity classes, DSMEM combine).  Within 1e-12 normalized of the direct FP64 result,
    including block 0 (zero prefix skipped), ragged tails and xcorr placement."""
    L, N, W_block = case
    rng = np.random.default_rng(N + L)
    s, k = rng.laplace(0, 0.2, L), rng.normal(0, 1 / np.sqrt(N), N)
    opts = pcb.opts_default(core=1)
    opts.fft_n = 16384
    with pcb.Plan(L, N, W_block, pcb.MODE_XCORR if mode == O.XCORR else pcb.MODE_CONV, pcb.PACK_FULL, 0,
                  opts=opts) as p:
        p.set_kernel(dev(k))
        info = p.info()
        assert info["fft_n"] == 16384
        r = torch.full((info["L_out"],), float("nan"), dtype=torch.float64, device=DEV)
        p.execute(dev(s), r)
        torch.cuda.synchronize()
        got = r.cpu().numpy()
    want = O.full_precision(s, k, mode=mode)
    assert not np.isnan(got).any()
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 1e-12


@pytest.mark.parametrize("packing,Q", [(O.ASYM2, 127), (O.ASYM2, 255), (O.ASYM3, 7), (O.SYM, 7), (O.SYM, 12)])
def test_fft_packed_exact_cfg3_geometry(packing, Q):
    """Config 3 geometry (N = 4096, W_block = 16384) on a 2^18-sample slice: the FFT core's
    packed outputs round to the exact integers (bit-exact dequantized outputs), residual
    monitor below 0.25 LSB.  asym2 at 8/9 bits is the config's operating point."""
    s, k = WL.cfg3(seed=0, L=1 << 18)
    ref = O.conv_pipeline(s, k, 16384, packing, Q, rmax_rule=O.RMAX_L1)
    assert ref.kernel.bound_ok and ref.mismatches == 0
    got, res, rc, info = fft_run(s, k, 16384, packing, Q)
    assert rc == pcb.PC_OK and res < 0.25, res
    assert np.array_equal(got, ref.out)


@pytest.mark.parametrize("packing", [O.SYM, O.ASYM2, O.FULL])
def test_fft_multi_part_blocks_and_xcorr(packing):
    """Blocks split into several FFT parts (large W_block, small transform) and xcorr mode."""
    rng = np.random.default_rng(3)
    s, q = rng.laplace(0, 0.3, 60000), rng.uniform(-1, 1, 700)
    Q = {O.SYM: 3, O.ASYM2: 63, O.FULL: 0}[packing]
    for mode in (O.CONV, O.XCORR):
        got, res, rc, info = fft_run(s, q, 16384, packing, Q, mode=mode)
        if packing == O.FULL:
            want = O.full_precision(s, q, mode)
            assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 1e-12
        else:
            ref = O.conv_pipeline(s, q, 16384, packing, Q, mode=mode, rmax_rule=O.RMAX_L1)
            assert rc == pcb.PC_OK and np.array_equal(got, ref.out)


@pytest.mark.parametrize("packing,Q", [(O.ASYM2, 63), (O.SYM, 3)])
def test_fft_batch_and_block_ranges(packing, Q):
    """FFT core with block peaks computed ahead (pc_block_peak): a 3-signal batch with padded
    strides (the peak buffer grows past the plan's one-signal size) and block ranges starting
    past block 0 (peaks indexed by absolute block), bit-exact against the oracle."""
    rng = np.random.default_rng(11)
    L, N, W_block = 70000, 700, 16384
    k = rng.uniform(-1, 1, N)
    S = rng.laplace(0, 0.3, (3, L))
    refs = [O.conv_pipeline(S[i], k, W_block, packing, Q, rmax_rule=O.RMAX_L1).out for i in range(3)]
    opts = pcb.opts_default(core=pcb.CORE_FFT, rmax_rule=O.RMAX_L1, bound_policy=pcb.BOUND_WARN)
    with pcb.Plan(L, N, W_block, pcb.MODE_CONV, PK[packing], Q, opts=opts) as p:
        p.set_kernel(dev(k))
        info = p.info()
        Lo = info["L_out"]
        Sd = torch.zeros((3, L + 5), dtype=torch.float64, device=DEV)
        Sd[:, :L] = dev(S)
        R = torch.full((3, Lo + 7), float("nan"), dtype=torch.float64, device=DEV)
        p.execute_batch(Sd, 3, L + 5, R, Lo + 7)
        torch.cuda.synchronize()
        for i in range(3):
            assert np.array_equal(R[i, :Lo].cpu().numpy(), refs[i]), i
        P = info["P"]
        out = np.full(Lo, np.nan)
        s_d = dev(S[1])
        for b0, b1 in [(0, 1), (1, P // 2), (P // 2, P)]:
            r = torch.full((Lo,), float("nan"), dtype=torch.float64, device=DEV)
            p.execute_blocks(s_d, 0, r, 0, b0, b1)
            torch.cuda.synchronize()
            got = r.cpu().numpy()
            sel = ~np.isnan(got)
            assert sel.any()
            out[sel] = got[sel]
        assert np.array_equal(out, refs[1])


def test_fft_residual_monitor_flags_overflowing_precision():
    """Fault injection: symmetric packing past its FFT precision (WARN policy) -> the monitor
    reports a residual above 0.25 LSB (PC_W_UNPACK_MARGIN) instead of silently passing."""
    s, k = WL.cfg3(seed=0, L=1 << 17)
    _, res_lo, rc_lo, _ = fft_run(s, k, 16384, O.SYM, 4)
    _, res_hi, rc_hi, _ = fft_run(s, k, 16384, O.SYM, 40)
    assert res_lo < 0.25 and rc_lo == pcb.PC_OK
    assert res_hi > res_lo and rc_hi == pcb.PC_W_UNPACK_MARGIN


def test_cfg3_full_size_fft_sampled():
    """Config 3 at full size through the FFT core: asym2 9-bit bit-exact on sampled blocks."""
    s, k = WL.cfg3(seed=0)
    geom = O.Geometry(len(s), len(k), 16384)
    blocks = sorted({0, 1, geom.P // 2, geom.P - 1})
    ref = O.conv_pipeline(s, k, 16384, O.ASYM2, 255, rmax_rule=O.RMAX_L1, blocks=blocks)
    got, res, rc, _ = fft_run(s, k, 16384, O.ASYM2, 255)
    sel = ~np.isnan(ref.out)
    assert rc == pcb.PC_OK and res < 0.25
    assert np.array_equal(got[sel], ref.out[sel])


@pytest.mark.parametrize("mode", [O.CONV, O.XCORR])
@pytest.mark.parametrize("packing", [O.FULL, O.SYM, O.ASYM2])
def test_execute_host_pipelined(mode, packing):
    """conv_execute_host over >= 128 blocks pipelines block ranges across copy streams;
    the result must equal the device-resident conv_execute bit for bit (same kernels,
    same block geometry, each output written once)."""
    rng = np.random.default_rng(7)
    L, N, W_block, Q = 600_001, 65, 1024, 127      # P = 627 blocks, ragged tail
    s = np.clip(rng.laplace(0.0, 0.2, L), -1.0, 1.0)
    k = rng.uniform(-1.0, 1.0, N)
    pk = {O.FULL: pcb.PACK_FULL, O.SYM: pcb.PACK_SYM, O.ASYM2: pcb.PACK_ASYM2}[packing]
    with pcb.Plan(L, N, W_block, pcb.MODE_XCORR if mode == O.XCORR else pcb.MODE_CONV, pk,
                  0 if packing == O.FULL else (31 if packing == O.SYM else Q),
                  rmax_rule=pcb.RMAX_L1) as p:
        p.set_kernel(dev(k))
        info = p.info()
        assert info["P"] >= 512
        r_dev = torch.empty(info["L_out"], dtype=torch.float64, device=DEV)
        p.execute(dev(s), r_dev)
        torch.cuda.synchronize()
        ref = r_dev.cpu().numpy()
        sh = torch.from_numpy(s).pin_memory()
        rh = torch.full((info["L_out"],), float("nan"), dtype=torch.float64).pin_memory()
        p.execute_host(sh, rh)
        assert np.array_equal(rh.numpy(), ref)
        rh2 = torch.full((info["L_out"],), float("nan"), dtype=torch.float64)   # pageable host memory
        p.execute_host(torch.from_numpy(s.copy()), rh2)
        assert np.array_equal(rh2.numpy(), ref)
    if packing == O.FULL and mode == O.CONV:
        full = O.full_precision(s, k)
        assert float(np.max(np.abs(ref - full)) / np.max(np.abs(full))) < 1e-12


@pytest.mark.parametrize("mode", [O.CONV, O.XCORR])
@pytest.mark.parametrize("case", [(50_000, 65, 1024, 20), (120_000, 129, 2048, 20), (60_000, 33, 512, 35)])
def test_literal_paper_unpack(mode, case):
    """conv_opts.unpack_form = UNPACK_LITERAL: the symmetric unpack follows the literal Eqs. (11)-(15) with
    the u_sys guard (PAPER eps, reading C6: exact for R_max < 89,524).  Its integers equal the
    exact integer convolution, so the output equals the oracle's literal-form pipeline and the
    balanced-digit output bit for bit."""
    L, N, W_block, Q = case
    rng = np.random.default_rng(L + N)
    s, k = np.clip(rng.laplace(0, 0.3, L), -1, 1), rng.uniform(-1, 1, N)
    Np = N | 1
    assert Np * Q * Q <= 52_000      # the u_sys guard is reliable well below 89,524 (none at 51k)
    ref = O.conv_pipeline(s, k, W_block, O.SYM, Q, mode=mode, eps_rule=O.EPS_PAPER, unpack_form="paper")
    assert ref.mismatches == 0
    opts = pcb.opts_default(eps_rule=EPS[O.EPS_PAPER], rmax_rule=O.RMAX_PAPER, bound_policy=pcb.BOUND_WARN)
    opts.unpack_form = pcb.UNPACK_LITERAL
    with pcb.Plan(L, N, W_block, pcb.MODE_XCORR if mode == O.XCORR else pcb.MODE_CONV, pcb.PACK_SYM, Q,
                  opts=opts) as p:
        p.set_kernel(dev(k))
        r = torch.full((p.info()["L_out"],), float("nan"), dtype=torch.float64, device=DEV)
        p.execute(dev(s), r)
        torch.cuda.synchronize()
        got = r.cpu().numpy()
    assert np.array_equal(got, ref.out)
    bal = O.conv_pipeline(s, k, W_block, O.SYM, Q, mode=mode, eps_rule=O.EPS_PAPER)
    assert np.array_equal(got, bal.out)


@pytest.mark.parametrize("packing,Q", [(O.FULL, 0), (O.SYM, 5), (O.ASYM2, 63)])
def test_xcorr_max_ties_lowest_lag(packing, Q):
    """Equal maxima at many lags (a periodic database signal and a query of whole periods):
    the score's lag is the lowest one (C17), across warp parts, jobs and blocks."""
    n_sig, L, N, per = 3, 50_000, 300, 100
    base = np.sin(2 * np.pi * np.arange(L) / per) * 0.5
    db = np.stack([base * (1 + 0.1 * i) for i in range(n_sig)])
    q = base[:N].copy()
    with pcb.Plan(L, N, 2048, pcb.MODE_XCORR, PK[packing], Q, rmax_rule=pcb.RMAX_L1) as p:
        p.set_kernel(dev(q))
        sc = torch.empty(n_sig, dtype=torch.float64, device=DEV)
        lag = torch.empty(n_sig, dtype=torch.int64, device=DEV)
        p.xcorr_max(dev(db), n_sig, L, sc, lag)
        torch.cuda.synchronize()
        sc, lag = sc.cpu().numpy(), lag.cpu().numpy()
    for i in range(n_sig):
        if packing == O.FULL:
            c = O.full_precision(db[i], q, O.XCORR)
            best = np.max(c)
            assert abs(sc[i] - best) <= 1e-12 * best and c[lag[i]] >= best * (1 - 1e-12)
        else:
            c = O.conv_pipeline(db[i], q, 2048, packing, Q, mode=O.XCORR, rmax_rule=O.RMAX_L1).out
            assert (sc[i], lag[i]) == O.xcorr_score(c)
            assert np.sum(c == sc[i]) > 1            # a real tie was resolved


@pytest.mark.parametrize("packing,Q", [(O.FULL, 0), (O.SYM, 3), (O.ASYM2, 32), (O.ASYM3, 5)])
def test_xcorr_pairs_per_pair_kernels(packing, Q):
    """NEXT-3 (§IV.C regime): block b of the left channel (zero-padded to all 2B-1 lags)
    cross-correlated with block b of the right channel, each right block companded as its own
    kernel (conv_plan_set_kernels; PAPER R_max so eps is common).  Per-pair score and lowest
    argmax equal the oracle pipeline run pair by pair; the lag recovers the channel delay."""
    B, delay = 1024, 17
    left, right = WL.stereo(seed=5, seconds=0.4, delay=delay)
    x, q = WL.stereo_pairs(left, right, B)
    n, L = x.shape
    with pcb.Plan(L, B, 4096, pcb.MODE_XCORR, PK[packing], Q, rmax_rule=pcb.RMAX_PAPER) as p:
        p.set_kernels(dev(q), n, B)
        sc = torch.empty(n, dtype=torch.float64, device=DEV)
        lag = torch.empty(n, dtype=torch.int64, device=DEV)
        p.xcorr_pairs(dev(x), n, L, sc, lag)
        torch.cuda.synchronize()
        sc, lag = sc.cpu().numpy(), lag.cpu().numpy()
    for i in range(n):
        if packing == O.FULL:
            c = O.full_precision(x[i], q[i], O.XCORR)
            best, j = O.xcorr_score(c)
            assert abs(sc[i] - best) <= 1e-12 * np.max(np.abs(c))
            assert c[lag[i]] >= best - 1e-12 * np.max(np.abs(c))
        else:
            ref = O.conv_pipeline(x[i], q[i], 4096, packing, Q, mode=O.XCORR, rmax_rule=O.RMAX_PAPER)
            assert ref.kernel.bound_ok and ref.mismatches == 0
            assert (sc[i], lag[i]) == O.xcorr_score(ref.out), i
    assert np.all(lag - (B - 1) == -delay)


# --------------------------------------------------------------------- DMMA core variants
@pytest.mark.parametrize("opt", ["prepack", "lookahead", "alu_pack", "fp64_pack", "fma_sym_auto"])
@pytest.mark.parametrize("packing", [O.SYM, O.ASYM2, O.ASYM3])
@pytest.mark.parametrize("mode", [O.CONV, O.XCORR])
def test_dmma_core_variants(opt, packing, mode):
    """The DMMA-core kernel's alternative schedules give bit-identical results: a2-a4 in a
    prepack kernel ahead of it (conv_opts.prepack = 1), a bounded producer claim-ahead
    (stage_cap = -2), integer-pipe companding and packing (pack_alu = 1, the default) or FP64
    ones (pack_alu = 2), and the auto core choice (DMMA, FMA for symmetric packing)."""
    L, N, W_block, Q = 90_000, 301, 4096, 31
    rng = np.random.default_rng(packing * 7 + mode)
    s, k = np.clip(rng.laplace(0, 0.3, L), -1, 1), rng.uniform(-1, 1, N)
    Q = min(Q, O.max_q_under_bound(None, N | 1, packing, O.EPS_POW2, O.RMAX_PAPER))
    ref = O.conv_pipeline(s, k, W_block, packing, Q, mode=mode)
    opts = pcb.opts_default(bound_policy=pcb.BOUND_WARN, exec=2)
    if opt == "prepack":
        opts.core_variant, opts.prepack = 2, 1
    elif opt == "lookahead":
        opts.core_variant, opts.stage_cap = 2, -2
    elif opt == "alu_pack":
        opts.core_variant, opts.pack_alu = 2, 1
    elif opt == "fp64_pack":
        opts.core_variant, opts.pack_alu = 2, 2
    with pcb.Plan(L, N, W_block, mode, PK[packing], Q, opts=opts) as p:
        p.set_kernel(dev(k))
        info = p.info()
        assert info["core_mma"] == (0 if (opt == "fma_sym_auto" and packing == O.SYM) else 1)
        r = torch.full((info["L_out"],), float("nan"), dtype=torch.float64, device=DEV)
        for _ in range(2):                       # twice: the queues / buffers are reused
            p.execute(dev(s), r)
        torch.cuda.synchronize()
    assert np.array_equal(r.cpu().numpy(), ref.out)


@pytest.mark.parametrize("mode", [O.CONV, O.XCORR])
@pytest.mark.parametrize("sig", ["uniform", "cfg2"])
def test_snr_calibration_matches_oracle(sig, mode):
    """conv_snr_calibrate (reading C18) against oracle.snr_calibration: the packed and
    full-precision outputs are the CUDA path's (bit-exact / 1e-12), the block statistics are
    bit-identical (C12), only the summation order of the four sums differs -- so the measured
    SNR, the model and the offset agree to 1e-9 dB; the offset then drives conv_adapt_block."""
    rng = np.random.default_rng(5 + mode)
    if sig == "uniform":
        s, k, W_block = rng.uniform(-128, 128, 1 << 16), rng.uniform(-128, 128, 401), 8192
    else:
        s, k = WL.cfg2(seed=3, L=1 << 17)
        W_block = 4096
    off, meas, model = O.snr_calibration(s, k, W_block, Q=8, packing=O.ASYM2, mode=mode)
    opts = pcb.opts_default(bound_policy=pcb.BOUND_WARN)
    with pcb.Plan(len(s), len(k), W_block, mode, PK[O.ASYM2], 8, opts=opts) as p:
        g_off, g_meas, g_model = p.snr_calibrate(dev(s), dev(k), 8)
    assert abs(g_meas - meas) < 1e-9 and abs(g_model - model) < 1e-9 and abs(g_off - off) < 1e-9
    if sig == "uniform":
        assert abs(g_off) < 1.0


@pytest.mark.parametrize("early", ["1", "0"])
@pytest.mark.parametrize("packing", [O.ASYM2, O.FULL])
def test_back_to_back_launches_early_fill(packing, early):
    """Consecutive tiled launches on one stream overlap (programmatic dependent launch): a
    launch's pipeline fill may start before the preceding one finished unless it reads what that
    one writes.  Chained (the second convolves the first's output, no sync in between): the
    host check must hold the fill back; independent inputs: it may run early.  Both bit-exact
    (full precision: the same bits as the unchained run)."""
    L, N, W_block, Q = 60_000, 129, 2048, 63
    rng = np.random.default_rng(17)
    s, k = np.clip(rng.laplace(0, 0.3, L), -1, 1), rng.uniform(-1, 1, N)
    Q = 0 if packing == O.FULL else Q
    ef = int(early)                                   # opt-in overlap of a launch's fill
    with pcb.Plan(L, N, W_block, O.CONV, PK[packing], Q, opts=pcb.opts_default(exec=2, early_fill=ef)) as p1, \
            pcb.Plan(L + N - 1, N, W_block, O.CONV, PK[packing], Q,
                     opts=pcb.opts_default(exec=2, early_fill=ef)) as p2:
        p1.set_kernel(dev(k))
        p2.set_kernel(dev(k))
        s_d = dev(s)
        r1 = torch.empty(L + N - 1, dtype=torch.float64, device=DEV)
        r2 = torch.empty(L + 2 * (N - 1), dtype=torch.float64, device=DEV)
        outs = []
        for _ in range(3):                            # chained, repeatedly, no host sync
            p1.execute(s_d, r1)
            p2.execute(r1, r2)
        torch.cuda.synchronize()
        got1, got2 = r1.cpu().numpy(), r2.cpu().numpy()
        s2 = np.clip(rng.laplace(0, 0.3, L), -1, 1)
        s2_d = dev(s2)
        ra, rb = torch.empty_like(r1), torch.empty_like(r1)
        for _ in range(3):                            # independent inputs back to back
            p1.execute(s_d, ra)
            p1.execute(s2_d, rb)
        torch.cuda.synchronize()
        got_a, got_b = ra.cpu().numpy(), rb.cpu().numpy()
    if packing == O.FULL:
        assert np.array_equal(got_a, got1)
        want2 = O.full_precision(O.full_precision(s, k), k)
        assert np.max(np.abs(got2 - want2)) / np.max(np.abs(want2)) < 1e-12
        return
    ref1 = O.conv_pipeline(s, k, W_block, packing, Q).out
    assert np.array_equal(got1, ref1) and np.array_equal(got_a, ref1)
    assert np.array_equal(got2, O.conv_pipeline(ref1, k, W_block, packing, Q).out)
    assert np.array_equal(got_b, O.conv_pipeline(s2, k, W_block, packing, Q).out)


def test_adaptive_step_graph_replay():
    """The adaptive step (a8 decisions + one tiled launch per packing) is stream-ordered device
    work only (the candidate table is uploaded once per kernel), so a CUDA graph of it replays
    with the eager result, for inputs whose decisions differ between replays."""
    s1, k = WL.cfg5(seed=1, L=1 << 17, N=1024)
    s2, _ = WL.cfg5(seed=2, L=1 << 17, N=1024)
    W_block, floor = 4096, 40.0
    with pcb.Plan(len(s1), len(k), W_block, pcb.MODE_CONV, pcb.PACK_ADAPTIVE, 0, rmax_rule=pcb.RMAX_L1) as p:
        p.set_kernel(dev(k))
        L_out = p.info()["L_out"]
        S = dev(s1)
        want = []
        for x in (s1, s2):
            r = torch.empty(L_out, dtype=torch.float64, device=DEV)
            p.adapt_block(dev(x), floor)
            p.execute(dev(x), r)
            torch.cuda.synchronize()
            want.append(r.cpu().numpy())
        R = torch.empty(L_out, dtype=torch.float64, device=DEV)
        gs = torch.cuda.Stream(DEV)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(gs):
            with torch.cuda.graph(graph, stream=gs):
                pcb.adapt_block(p.h, S, floor, 0.0, None, gs.cuda_stream)
                pcb.execute(p.h, S, R, gs.cuda_stream)
        for x, w in ((s1, want[0]), (s2, want[1]), (s1, want[0])):
            S.copy_(dev(x))
            R.fill_(float("nan"))
            torch.cuda.synchronize()
            graph.replay()
            torch.cuda.synchronize()
            assert np.array_equal(R.cpu().numpy(), w)


@pytest.mark.parametrize("packing,Q", [(O.ASYM2, 127), (O.ASYM2, 63), (O.SYM, 5)])   # R within each bound
def test_fft_core_backend_validation_worst_case(packing, Q):
    """Backend validation of the GPU FFT core (the u_sys guard's purpose, P:103,
    P:153): worst-case packed operands -- every sample and tap at full magnitude (+-1, so
    every companded digit is +-S_q / +-K_q) -- over 100 random sign patterns in 4 launches at
    the cfg3 geometry; the core's last-digit deviation (the residual monitor) stays below
    0.5 LSB, so the integers equal the exact direct core's bit for bit, and u_sys calibrated
    as 4 x the measured absolute deviation is reported next to the paper's value."""
    rng = np.random.default_rng(Q)
    L, N, W_block = 1 << 17, 4096, 16384
    worst = 0.0
    for _ in range(4):
        s = rng.choice([-1.0, 1.0], L)
        k = rng.choice([-1.0, 1.0], N)
        got, res, rc, info = fft_run(s, k, W_block, packing, Q)
        ref = gpu_run(s, k, W_block, packing, Q, rmax_rule=O.RMAX_L1, debug=False)["r"]
        assert np.array_equal(got, ref)
        assert res < 0.5
        worst = max(worst, res)
    u_sys = 4.0 * worst * info["eps"]              # absolute deviation of a packed core output
    print(f"FFT core {packing} Q={Q}: max last-digit residual {worst:.3g} LSB, calibrated u_sys {u_sys:.3g} "
          f"(paper {O.U_SYS_PAPER:.4g})")


@pytest.mark.parametrize("packing,N,mma", [(O.SYM, 513, 0), (O.SYM, 2049, 1), (O.ASYM3, 129, 0), (O.ASYM3, 513, 1),
                                           (O.ASYM2, 129, 1), (O.FULL, 129, 1)])
def test_auto_core_choice(packing, N, mma):
    """The auto core rule (conv_opts.core_variant = 0): DMMA except short symmetric (< 768 core taps)
    and asym3 (< 256) cores, which keep the FMA loop -- the measured crossovers."""
    W_block = 8192
    with pcb.Plan(100_000, N, W_block, pcb.MODE_CONV, PK[packing], 0 if packing == O.FULL else 3,
                  opts=pcb.opts_default(bound_policy=pcb.BOUND_WARN)) as p:
        p.set_kernel(dev(np.linspace(-1, 1, N)))
        info = p.info()
        assert info["core_mma"] == mma and info["core_tile"] in (12, 14, 16)


# --------------------------------------------------------------------- round 2: boundary (§8(b))
def fft_plan(L, k, packing, Q, policy, fft_n=0, W_block=16384, mode=O.CONV):
    opts = pcb.opts_default(core=pcb.CORE_FFT, rmax_rule=pcb.RMAX_L1, bound_policy=policy, fft_n=fft_n)
    p = pcb.Plan(L, len(k), W_block, mode, PK[packing], Q, opts=opts)
    try:
        p.set_kernel(dev(k))
    except Exception:
        p.close()
        raise
    return p


def test_fft_backend_validation_at_set_kernel():
    """conv_plan_set_kernel validates FFT-core plans: at the cfg3 geometry
    asym2 up to Q = 191 (~8.6 bits) passes -- 4 x the worst last-digit residual <= 0.5 LSB --
    with a calibrated u_sys; asym2 Q = 285, within its R_max bound (L1 rule), has a worst-case
    residual near 0.3-0.4 LSB and is refused under STRICT (PC_E_BACKEND, kernel not installed)
    and accepted under WARN (backend_ok = 0), where executing worst-case data makes the runtime
    monitor fire (PC_W_UNPACK_MARGIN from conv_execute and conv_plan_residual)."""
    s, k = WL.cfg3(seed=0, L=1 << 18)
    for Q in (63, 127, 191):
        with fft_plan(len(s), k, O.ASYM2, Q, pcb.BOUND_STRICT) as p:
            info = p.info()
            assert info["bound_ok"] == 1 and info["backend_ok"] == 1
            assert 0.0 < info["backend_resid"] <= 0.125 and info["u_sys_cal"] > 0.0
            print(f"validated asym2 Q={Q}: resid {info['backend_resid']:.4g} LSB, u_sys {info['u_sys_cal']:.4g}")
    with pytest.raises(pcb.PcError) as ei:
        fft_plan(len(s), k, O.ASYM2, 285, pcb.BOUND_STRICT, fft_n=4096)
    assert ei.value.code == pcb.PC_E_BACKEND
    L = 1 << 20
    with fft_plan(L, k, O.ASYM2, 285, pcb.BOUND_WARN, fft_n=4096) as p:
        info = p.info()
        assert info["bound_ok"] == 1 and info["backend_ok"] == 0 and info["backend_resid"] > 0.125
        x = dev(np.where(np.random.default_rng(1).random(L) < 0.5, -1.0, 1.0))
        r = torch.empty(info["L_out"], dtype=torch.float64, device=DEV)
        p.execute(x, r)
        torch.cuda.synchronize()
        with pytest.warns(pcb.UnpackMarginWarning):
            rc = p.execute(x, r)                  # the completed launch raised the host-mapped flag
        assert rc == pcb.PC_W_UNPACK_MARGIN
        torch.cuda.synchronize()
        res, rc = p.residual(reset=True)
        assert rc == pcb.PC_W_UNPACK_MARGIN and res > 0.25
        assert p.execute(x * 0.0, r) == pcb.PC_OK  # flag cleared by the reset


def test_direct_plans_skip_backend_validation():
    s, k = WL.cfg2(seed=0, L=1 << 16)
    with pcb.Plan(len(s), len(k), 4096, pcb.MODE_CONV, pcb.PACK_ASYM2, 511, rmax_rule=pcb.RMAX_L1) as p:
        p.set_kernel(dev(k))
        info = p.info()
        assert info["backend_ok"] == -1 and info["u_sys_cal"] == 0.0


@pytest.mark.parametrize("eps_rule,exact", [(O.EPS_POW2, True), (O.EPS_PAPER, False)])
def test_debug_max_residual(eps_rule, exact):
    """conv_execute_debug's max_residual (§8(b)): exactly 0 under the dyadic eps (C4: every
    packed product exact); under the paper's eps (Eq. (6)) a rounding residual below 0.5 LSB."""
    rng = np.random.default_rng(9)
    L, N, W_block, Q = 30000, 65, 1024, 20
    s, k = np.clip(rng.laplace(0, 0.3, L), -1, 1), rng.uniform(-1, 1, N)
    opts = pcb.opts_default(eps_rule=EPS[eps_rule], bound_policy=pcb.BOUND_WARN, exec=pcb.EXEC_PERBLOCK)
    ref = O.conv_pipeline(s, k, W_block, O.SYM, Q, eps_rule=eps_rule)
    with pcb.Plan(L, N, W_block, pcb.MODE_CONV, pcb.PACK_SYM, Q, opts=opts) as p:
        p.set_kernel(dev(k))
        r = torch.empty(p.info()["L_out"], dtype=torch.float64, device=DEV)
        res = p.execute_debug(dev(s), r, max_residual=True)
        assert np.array_equal(r.cpu().numpy(), ref.out)
    if exact:
        assert res == 0.0
    else:
        assert 0.0 < res < 0.5


def test_binding_rejects_bad_device_buffers():
    """No lengths cross the C ABI, so the binding refuses wrong dtype / short / strided / host
    buffers before any launch (PC_E_CONFIG)."""
    s, k = WL.cfg1(seed=0, L=8192)
    with pcb.Plan(len(s), len(k), 1024, pcb.MODE_CONV, pcb.PACK_ASYM2, 127) as p:
        p.set_kernel(dev(k))
        Lo = p.info()["L_out"]
        good_s, good_r = dev(s), torch.empty(Lo, dtype=torch.float64, device=DEV)
        bad = [(good_s.float(), good_r), (good_s[:-1], good_r), (good_s, good_r[:-1]),
               (torch.empty(2 * len(s), dtype=torch.float64, device=DEV)[::2], good_r),
               (torch.from_numpy(s), good_r)]
        for a, b in bad:
            with pytest.raises(pcb.PcError) as ei:
                p.execute(a, b)
            assert ei.value.code == pcb.PC_E_CONFIG
        with pytest.raises(pcb.PcError):
            p.execute(good_s, good_s)                 # in place: s and r overlap
        with pytest.raises(pcb.PcError):
            p.set_kernel(dev(k[:-1]))
        assert p.execute(good_s, good_r) == pcb.PC_OK


@pytest.mark.parametrize("floor", [35.0, 65.0])      # sym + asym2 blocks; asym2 + full blocks
def test_adaptive_block_lists_many_blocks(floor):
    """pc_adapt_lists' compaction across warps and rounds (P > 4096 blocks, two packings
    interleaved per floor): every output is written (NaN-filled buffer) and equals the oracle's adaptive
    pipeline (packed blocks bit-exact, full-precision blocks within 1e-12)."""
    rng = np.random.default_rng(11)
    N, W_block = 33, 128                              # W = 94: P = 5200 blocks
    P = 5200
    L = P * 94
    scale = np.repeat(10.0 ** rng.uniform(-2, 0, P + 1), 94)[:L]
    s = rng.laplace(0, 1.0, L) * scale
    k = rng.normal(0, 1 / np.sqrt(N), N)
    y_ref, dec_ref, qmode = O.adaptive_pipeline(s, k, W_block, floor)
    modes = {m for m, _, _ in dec_ref}
    assert len(modes) >= 2, modes
    with pcb.Plan(L, N, W_block, pcb.MODE_CONV, pcb.PACK_ADAPTIVE, 0, rmax_rule=pcb.RMAX_L1) as p:
        p.set_kernel(dev(k))
        info = p.info()
        assert info["P"] > 4096
        s_d = dev(s)
        dec = p.adapt_block(s_d, floor)
        assert [(d[0], d[1]) for d in dec] == [(PK[m], q) for m, q, _ in dec_ref]
        r = torch.full((info["L_out"],), float("nan"), dtype=torch.float64, device=DEV)
        p.execute(s_d, r)
        torch.cuda.synchronize()
        got = r.cpu().numpy()
    assert not np.isnan(got).any()
    geom = O.Geometry(L, N, W_block)
    for w, (m, q, _) in enumerate(dec_ref):
        g0 = geom.block_start(w)
        o0, n_out = geom.kept(w)
        lo, hi = g0 + o0, min(g0 + o0 + n_out, geom.L_out)
        if m == O.FULL:
            scl = max(np.max(np.abs(y_ref[lo:hi])), 1e-300)
            assert np.max(np.abs(got[lo:hi] - y_ref[lo:hi])) / scl < 1e-12, w
        else:
            assert np.array_equal(got[lo:hi], y_ref[lo:hi]), w


@pytest.mark.parametrize("mode", [O.CONV, O.XCORR])
def test_execute_host_blocks_shards(mode):
    """conv_execute_host_blocks (a rank's shard through host buffers): the shards'
    host outputs assemble to the oracle's output bit for bit (pipelined and one-pass ranges)."""
    rng = np.random.default_rng(21)
    L, N, W_block, Q = 300_000, 129, 1024, 127
    s, k = rng.laplace(0, 0.2, L), rng.uniform(-1, 1, N)
    ref = O.conv_pipeline(s, k, W_block, O.ASYM2, Q, mode=mode)
    with pcb.Plan(L, N, W_block, mode, pcb.PACK_ASYM2, Q) as p:
        p.set_kernel(dev(k))
        info = p.info()
        for G in (1, 2, 5):
            out = np.full(info["L_out"], np.nan)
            for rank in range(G):
                sh = pcb.shard_range(L, N, W_block, mode, rank, G)
                sh_h = torch.from_numpy(s[sh["in_begin"]:sh["in_end"]].copy()).pin_memory()
                rh = torch.full((max(1, sh["out_end"] - sh["out_begin"]),), float("nan"), dtype=torch.float64)
                assert p.execute_host_blocks(sh_h, sh["in_begin"], rh, sh["out_begin"], sh["block_begin"],
                                             sh["block_end"]) == pcb.PC_OK
                out[sh["out_begin"]:sh["out_end"]] = rh.numpy()[:sh["out_end"] - sh["out_begin"]]
            assert np.array_equal(out, ref.out), G


def test_adapt_blocks_shards_equal_whole():
    """conv_adapt_blocks + conv_execute_blocks on block-range shards (cfg5's multi-GPU split):
    every shard's decisions equal the whole-signal decisions of its blocks, and the assembled
    output is bit-identical to the single adaptive run."""
    s, k = WL.cfg5(seed=2, L=1 << 18, N=1024)
    W_block, floor = 4096, 40.0
    L, N = len(s), len(k)
    with pcb.Plan(L, N, W_block, pcb.MODE_CONV, pcb.PACK_ADAPTIVE, 0, rmax_rule=pcb.RMAX_L1) as p:
        p.set_kernel(dev(k))
        info = p.info()
        s_d = dev(s)
        whole = p.adapt_block(s_d, floor)
        r = torch.empty(info["L_out"], dtype=torch.float64, device=DEV)
        p.execute(s_d, r)
        torch.cuda.synchronize()
        want = r.cpu().numpy()
        for G in (2, 3):
            out = np.full(info["L_out"], np.nan)
            for rank in range(G):
                sh = pcb.shard_range(L, N, W_block, 0, rank, G)
                xs = dev(s[sh["in_begin"]:sh["in_end"]])
                dec = p.adapt_blocks(xs, sh["in_begin"], sh["block_begin"], sh["block_end"], floor, want=True)
                assert dec == whole[sh["block_begin"]:sh["block_end"]]
                n = sh["out_end"] - sh["out_begin"]
                rs = torch.full((max(1, n),), float("nan"), dtype=torch.float64, device=DEV)
                p.execute_blocks(xs, sh["in_begin"], rs, sh["out_begin"], sh["block_begin"], sh["block_end"])
                torch.cuda.synchronize()
                out[sh["out_begin"]:sh["out_end"]] = rs.cpu().numpy()[:n]
                with pytest.raises(pcb.PcError) as ei:       # blocks outside the decided range
                    p.execute(s_d, r)
                assert ei.value.code == pcb.PC_E_STATE
            assert np.array_equal(out, want), G


def test_best_match_kernel():
    """conv_best_match (the database winner, C17): largest score, ties to the smallest index,
    over per-signal arrays and over gathered candidate rows."""
    rng = np.random.default_rng(4)
    n = 3000
    sc = np.round(rng.normal(0, 1, n), 1)                  # many ties
    lg = rng.integers(0, 1 << 20, n)
    best = torch.empty(3, dtype=torch.float64, device=DEV)
    pcb.best_match(best, n, score_dev=dev(sc), lag_dev=dev(lg), first_index=77)
    i = int(np.flatnonzero(sc == sc.max())[0])
    assert best.cpu().tolist() == [sc[i], float(lg[i]), float(77 + i)]
    cand = np.array([[1.0, 5, 9], [2.0, 6, 4], [2.0, 7, 3], [-1.0, 8, 0]])
    pcb.best_match(best, 4, cand_dev=dev(cand.reshape(-1)))
    assert best.cpu().tolist() == [2.0, 7.0, 3.0]


# --------------------------------------------------------------------- randomized geometry sweep
def _random_case(rng):
    """A random valid geometry and operating point: N in [1, 700] (odd and even), W_block from
    the smallest valid (W = 2N') to 8x that, L from one sample to ~30 blocks, every packing, the
    largest Q its bound allows (or a smaller random one), both companding-range rules and both
    modes; signals of several distributions (Laplace, uniform, sparse, constant runs)."""
    N = int(rng.integers(1, 700))
    Np = N | 1
    W = 2 * Np + 2 * int(rng.integers(0, 4 * Np))
    W_block = W + Np + 1
    L = int(rng.integers(1, 30 * W))
    mode = int(rng.integers(0, 2))
    if mode == O.XCORR and L < N:
        L = N + int(rng.integers(0, W))
    packing = [O.SYM, O.ASYM2, O.ASYM3][int(rng.integers(0, 3))]
    rmax = [O.RMAX_PAPER, O.RMAX_L1][int(rng.integers(0, 2))]
    kind = int(rng.integers(0, 4))
    if kind == 0:
        s = np.clip(rng.laplace(0, 0.3, L), -1, 1)
    elif kind == 1:
        s = rng.uniform(-1, 1, L)
    elif kind == 2:
        s = rng.normal(0, 1, L) * (rng.random(L) < 0.05)
    else:
        s = np.repeat(rng.uniform(-1, 1, L // 64 + 1), 64)[:L]
    k = rng.normal(0, 1, N) if rng.random() < 0.5 else rng.uniform(-1, 1, N)
    kp = np.zeros(Np)
    kp[:N] = k[::-1] if mode == O.XCORR else k
    qmax = O.max_q_under_bound(kp, Np, packing, O.EPS_POW2, rmax, q_cap=4096)
    Q = qmax if rng.random() < 0.6 else max(1, int(rng.integers(1, qmax + 1)))
    return s, k, W_block, packing, Q, rmax, mode


@pytest.mark.parametrize("seed", range(96))
def test_randomized_geometries_bit_exact(seed):
    """96 random (L, N, W_block, packing, Q, range rule, mode, signal) cases through the
    production path (auto core and execution form) and, for every third case, the forced FMA
    core / per-block kernel: the dequantized outputs equal the oracle's bit for bit, and the
    integers are exact (the oracle's own self-check)."""
    rng = np.random.default_rng(1000 + seed)
    s, k, W_block, packing, Q, rmax, mode = _random_case(rng)
    if Q < 1:
        pytest.skip("no Q meets the bound")
    ref = O.conv_pipeline(s, k, W_block, packing, Q, mode=mode, rmax_rule=rmax)
    assert ref.mismatches == 0
    variants = [dict()]
    if seed % 3 == 0:
        variants += [dict(core_variant=pcb.CORE_FMA, exec=pcb.EXEC_TILED), dict(exec=pcb.EXEC_PERBLOCK)]
    for v in variants:
        opts = pcb.opts_default(rmax_rule=rmax, **v)
        try:
            with pcb.Plan(len(s), len(k), W_block, mode, PK[packing], Q, opts=opts) as p:
                p.set_kernel(dev(k))
                r = torch.full((p.info()["L_out"],), float("nan"), dtype=torch.float64, device=DEV)
                p.execute(dev(s), r)
                torch.cuda.synchronize()
        except pcb.PcError as ex:                      # a forced form may not fit (shared memory)
            assert ex.code == pcb.PC_E_CONFIG and v, ex
            continue
        assert np.array_equal(r.cpu().numpy(), ref.out), (seed, v, len(s), len(k), W_block, packing, Q, rmax, mode)


@pytest.mark.parametrize("packing,Q", [(O.ASYM2, 511), (O.SYM, 22), (O.ASYM3, 22), (O.FULL, 0)])
@pytest.mark.parametrize("raw", [0, 1, 2])
def test_raw_staged_producers_bit_exact(packing, Q, raw):
    """The persistent kernel's raw-staged producers (opts.raw_staging: 0 auto -- asym2 and sym --,
    1 forced, 2 off): the block arrives by one TMA bulk copy with the head element (input not
    16-byte aligned) and an odd tail loaded by threads.  A ragged length, block-range launches
    (b0 > 0) and a misaligned input pointer, bit-exact against the oracle in every form."""
    rng = np.random.default_rng(77)
    L, N, W_block = 61_117, 513, 4096
    s, k = rng.laplace(0, 0.25, L), rng.uniform(-1, 1, N)
    ref = O.conv_pipeline(s, k, W_block, packing, Q, rmax_rule=O.RMAX_L1).out

    def same(got):                                    # full precision: FP64 rounding order (C16)
        if packing == O.FULL:
            return np.max(np.abs(got - ref)) / np.max(np.abs(ref)) < 1e-12
        return np.array_equal(got, ref)

    opts = pcb.opts_default(rmax_rule=O.RMAX_L1, raw_staging=raw)
    with pcb.Plan(L, N, W_block, pcb.MODE_CONV, PK[packing], Q, opts=opts) as p:
        p.set_kernel(dev(k))
        info = p.info()
        buf = torch.zeros(L + 1, dtype=torch.float64, device=DEV)
        buf[1:] = dev(s)
        for src in (dev(s), buf[1:]):
            r = torch.full((info["L_out"],), float("nan"), dtype=torch.float64, device=DEV)
            p.execute(src, r)
            torch.cuda.synchronize()
            assert same(r.cpu().numpy()), (raw, src.data_ptr() % 16)
        out = np.full(info["L_out"], np.nan)
        P = info["P"]
        for b0, b1 in [(0, 3), (3, P // 2), (P // 2, P)]:
            r = torch.full((info["L_out"],), float("nan"), dtype=torch.float64, device=DEV)
            p.execute_blocks(buf[1:], 0, r, 0, b0, b1)
            torch.cuda.synchronize()
            got = r.cpu().numpy()
            sel = ~np.isnan(got)
            out[sel] = got[sel]
        assert same(out)
