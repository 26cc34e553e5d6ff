"""Pins of the CPU oracle against things other than itself (task rule ③): the paper's
printed values (tests/golden/paper_values.json, each with its citation), SPEC.md worked
examples, brute-force pure-Python convolution on tiny inputs, exhaustive small sweeps,
closed forms and invariants.  No GPU needed."""
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle as O
from paper_1201_3018_b200 import workloads as WL

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def brute_conv(a, b):
    """Eq. (1) written out: r[m] = sum_n a[m-n] b[n], pure Python integers/floats."""
    a, b = list(a), list(b)
    out = []
    for m in range(len(a) + len(b) - 1):
        acc = 0
        for n in range(len(b)):
            if 0 <= m - n < len(a):
                acc += a[m - n] * b[n]
        out.append(acc)
    return out


# --------------------------------------------------------------------------- rounding / companding

def test_rhaz_ties_and_near_ties():
    x = np.array([2.5, -2.5, 0.5, -0.5, 1.4999999999999998, 0.49999999999999994, -0.49999999999999994,
                  3.0, -0.0, 1e300, 4503599627370495.5])
    got = O.rhaz(x)
    want = [3, -3, 1, -1, 1, 0, 0, 3, 0, 1e300, 4503599627370496.0]
    assert list(got) == want


@pytest.mark.parametrize("ex", GOLD["compand_examples"])
def test_compand_spec_examples(ex):
    s, c, peak = O.compand(ex["x"], ex["Q"])
    assert list(s) == ex["s"]
    if "c" in ex:
        assert c == ex["c"] and peak == ex["peak"]


def test_compand_invariants():
    rng = np.random.default_rng(5)
    for Q in (1, 7, 127, 511):
        x = rng.laplace(0, 0.3, 5000)
        s, c, p = O.compand(x, Q)
        assert np.max(np.abs(s)) == Q                       # peak maps to +-Q exactly
        assert np.all(np.abs(c * x - s) <= 0.5)
        assert np.all(s == np.round(s))


# --------------------------------------------------------------------------- eps / bounds

@pytest.mark.parametrize("ex", GOLD["eps_paper_examples"])
def test_eps_paper_examples(ex):
    e = O.packing_coefficient(ex["R"], O.EPS_PAPER)
    if "eps" in ex:
        assert e.eps == ex["eps"]
    if "eps_inv" in ex:
        assert e.eps_inv == ex["eps_inv"]


def test_eps_pow2_and_radix():
    for R in (1, 2, 3, 18, 1000, 131071, 67108863):
        e = O.packing_coefficient(R, O.EPS_POW2)
        assert e.eps_inv == 2.0 ** e.b and e.eps * e.eps_inv == 1.0
        assert 2 * R + 1 <= e.eps_inv < 2 * (2 * R + 1)     # smallest power of two >= 2R+1
        r = O.packing_coefficient(R, O.EPS_RADIX)
        assert r.eps_inv == 2 * R + 1


def test_table1_bounds_and_pow2_algebra():
    assert O.BOUND_TABLE1[O.SYM] == GOLD["bound_sym"]["value"]
    assert O.BOUND_TABLE1[O.ASYM3] == GOLD["bound_asym3"]["value"]
    assert O.BOUND_TABLE1[O.ASYM2] == GOLD["bound_asym2"]["value"]
    # POW2 exactness bounds, re-derived here in plain integers (reading C4)
    R3, R2 = 2 ** 17 - 1, 2 ** 26 - 1
    assert R3 * (2 ** 36 + 2 ** 18 + 1) < 2 ** 53 and (R3 + 1) * (2 ** 38 + 2 ** 19 + 1) >= 2 ** 53
    assert R2 * (2 ** 27 + 1) < 2 ** 53 and (R2 + 1) * (2 ** 28 + 1) >= 2 ** 53
    assert O.pow2_bound(O.SYM) == R3 == O.pow2_bound(O.ASYM3)
    assert O.pow2_bound(O.ASYM2) == R2
    # Table 1's bounds are the mantissa budget (2R)^M ~ 2^52.7
    assert abs(3 * math.log2(2 * 97667) - 52.727) < 0.01
    assert abs(2 * math.log2(2 * 43165096) - 52.727) < 0.01


# --------------------------------------------------------------------------- packing

@pytest.mark.parametrize("ex", GOLD["pack_sym_signal_examples"])
def test_pack_sym_signal_examples(ex):
    got = O.pack_symmetric_signal(ex["s"], ex["eps"])
    assert np.allclose(got, ex["packed"], rtol=0, atol=1e-15)


def test_pack_sym_kernel_reading_c1():
    ex = GOLD["pack_sym_kernel_example"]
    assert list(O.pack_symmetric_kernel(ex["k"], ex["eps_inv"])) == ex["packed_C1"]


def test_pack_asym_spec_example():
    # s~=[1..6], M=2, W=4 (segment stride 2), eps=0.1 -> [1.3, 2.4, 3.5]: with our
    # reading C8 a segment q word i is s_loc[o0 + qS - (N'-1) + i]; o0=N'-1, S=2 reproduces it.
    got = O.pack_asymmetric_signal([1, 2, 3, 4, 5, 6], 0.1, 2, o0=0, S=2, Np=1)
    assert np.allclose(got, [1 + 0.1 * 3, 2 + 0.1 * 4], atol=1e-15)


# --------------------------------------------------------------------------- unpacking pins

def _sym_roundtrip(s, k, eps, eps_inv, R, form):
    sbar = O.pack_symmetric_signal(s, eps)
    kbar = O.pack_symmetric_kernel(k, eps_inv)
    rbar = np.convolve(sbar, kbar)
    if form == "balanced":
        A, B, C = O.unpack_balanced_sym(rbar, eps_inv)
        r = O.assemble_sym(A, B, C, first_is_seed=False)
    else:
        even, odd = O.unpack_paper_sym(rbar, R, eps, eps_inv, O.U_SYS_PAPER, 0)
        r = np.empty(2 * rbar.shape[0])
        r[0::2], r[1::2] = even, odd
    n = len(s) + len(k) - 1
    return [int(v) for v in r[:n]], r[n:]


@pytest.mark.parametrize("form", ["balanced", "paper"])
def test_spec_s300_worked_example(form):
    ex = GOLD["unpack_sym_example"]
    want = brute_conv(ex["s"], ex["k"])
    assert want == [2, -5, 7, -7, 4, 0, -5, 7, -4, 1]
    got, tail = _sym_roundtrip(ex["s"], ex["k"], 1.0 / ex["eps_inv"], float(ex["eps_inv"]), ex["R"], form)
    assert got == want
    assert np.all(tail == 0)


def test_printed_eq5_fails_s300():
    """Reading C1: the printed Eq. (5) parity gives no convolution output."""
    ex = GOLD["unpack_sym_example"]
    k = np.array(ex["k"] + [0], dtype=float)
    kbar_printed = k[0::2] + ex["eps_inv"] * k[1::2]
    rbar = np.convolve(O.pack_symmetric_signal(ex["s"], 1 / 36), kbar_printed)
    A, B, C = O.unpack_balanced_sym(rbar, 36.0)
    r = O.assemble_sym(A, B, C, first_is_seed=False)[:10]
    assert [int(v) for v in r] != brute_conv(ex["s"], ex["k"])


def _exhaustive_sym(eps_rule, q=2, ns=4, nk=3):
    vals = range(-q, q + 1)
    sigs = [np.array(s, float) for s in itertools.product(vals, repeat=ns)]
    fails, fails_without_plusR = 0, 0
    R = nk * q * q
    e = O.packing_coefficient(R, eps_rule)
    sbars = [O.pack_symmetric_signal(s, e.eps) for s in sigs]
    for k in itertools.product(vals, repeat=nk):
        kbar = O.pack_symmetric_kernel(np.array(k, float), e.eps_inv)
        for s, sbar in zip(sigs, sbars):
            rbar = np.convolve(sbar, kbar)
            A, B, C = O.unpack_balanced_sym(rbar, e.eps_inv)
            got = O.assemble_sym(A, B, C, False)[:ns + nk - 1]
            want = np.array(brute_conv(s.astype(int), k), float)
            if not np.array_equal(got, want):
                fails += 1
                # every PAPER-eps failure involves a +R_max partial (reading C2)
                sb = s.astype(int)
                part = [sum(sb[2 * m - 2 * n] * k[2 * n] for n in range(2) if 0 <= 2 * m - 2 * n < ns and 2 * n < nk)
                        for m in range(3)]
                if R not in want and R not in part and R not in [int(v) for v in A]:
                    fails_without_plusR += 1
    return fails, fails_without_plusR


@pytest.mark.slow
def test_exhaustive_sym_radix_and_pow2_exact():
    """Exhaustive s~ in [-2,2]^4, k~ in [-2,2]^3 (78,125 pairs): zero mismatches (C2/C4)."""
    assert _exhaustive_sym(O.EPS_POW2)[0] == 0
    assert _exhaustive_sym(O.EPS_RADIX)[0] == 0


@pytest.mark.slow
def test_exhaustive_sym_paper_eps_plus_rmax_carry():
    """Eq. (6)'s radix 2R_max cannot hold +R_max (reading C2): failures exist, and every
    one of them involves a digit equal to +R_max."""
    fails, other = _exhaustive_sym(O.EPS_PAPER)
    assert fails > 0 and other == 0


def test_asym_spec_examples():
    ex = GOLD["unpack_asym_example"]
    eps = 1.0 / ex["eps_inv"]
    v = ex["t"][0] + eps * ex["t"][1]
    for ts in (O.unpack_balanced_asym(np.array([v]), float(ex["eps_inv"]), 2),
               O.unpack_floor_asym(np.array([v]), ex["R"], eps, float(ex["eps_inv"]), 2)):
        assert [int(t[0]) for t in ts] == ex["t"]


def test_asym_worst_case_s311():
    """M=3, all t_q = +R_max -> exact recovery; holds for radix >= 2R+1 only (C2)."""
    R = GOLD["unpack_asym_worst"]["R"]
    for rule, exact in ((O.EPS_RADIX, True), (O.EPS_POW2, True), (O.EPS_PAPER, False)):
        e = O.packing_coefficient(R, rule)
        v = R + e.eps * (R + e.eps * R)
        fl = [int(t[0]) for t in O.unpack_floor_asym(np.array([v]), R, e.eps, e.eps_inv, 3)]
        assert (fl == [R, R, R]) == exact, (rule, fl)
        if rule != O.EPS_PAPER:
            bal = [int(t[0]) for t in O.unpack_balanced_asym(np.array([v]), e.eps_inv, 3)]
            assert bal == [R, R, R]


def test_asym_random_digits_roundtrip():
    rng = np.random.default_rng(1)
    for M in (2, 3):
        for R in (3, 18, 1000, 131071 if M == 3 else 67108863):
            e = O.packing_coefficient(R, O.EPS_POW2)
            t = rng.integers(-R, R + 1, (M, 2000)).astype(float)
            t[:, :5] = R                   # saturating
            t[:, 5:10] = -R
            v = t[M - 1].copy()
            for q in range(M - 2, -1, -1):
                v = t[q] + e.eps * v
            got = O.unpack_balanced_asym(v, e.eps_inv, M)
            assert all(np.array_equal(g, tt) for g, tt in zip(got, t))


def test_literal_unpack_guard_limit():
    """Reading C6: literal Eqs. (11)-(15) work at moderate R; the u_sys guard shifts
    the side-eps digit by u_sys eps^-2 >= 1 beyond R = 1/(2 sqrt(u_sys)) = 89,524."""
    assert int(1 / (2 * math.sqrt(O.U_SYS_PAPER))) == 89524
    rng = np.random.default_rng(3)
    s = rng.integers(-4, 5, 64).astype(float)
    k = rng.integers(-4, 5, 9).astype(float)
    R = 9 * 16
    e = O.packing_coefficient(R, O.EPS_PAPER)
    got, _ = _sym_roundtrip(s, k, e.eps, e.eps_inv, R, "paper")
    want = brute_conv(s.astype(int), k.astype(int))
    # +R_max outputs may carry under the paper's eps (C2); this input has none
    assert R not in want
    assert got == want


# --------------------------------------------------------------------------- pipeline pins

def _int_case(seed, L, N, W_block, Q):
    rng = np.random.default_rng(seed)
    s = rng.uniform(-1, 1, L)
    k = rng.uniform(-1, 1, N)
    return s, k


@pytest.mark.parametrize("packing", [O.SYM, O.ASYM2, O.ASYM3])
@pytest.mark.parametrize("eps_rule", [O.EPS_POW2, O.EPS_RADIX])
@pytest.mark.parametrize("L,N,W_block", [(1000, 9, 40), (777, 10, 34), (50, 3, 12), (5, 1, 4), (3000, 33, 110)])
def test_pipeline_integer_exact_vs_brute_force(packing, eps_rule, L, N, W_block):
    s, k = _int_case(L + N, L, N, W_block, 7)
    Q = 7
    res = O.conv_pipeline(s, k, W_block, packing, Q, eps_rule=eps_rule, keep_blocks=True)
    assert res.kernel.bound_ok
    assert res.mismatches == 0
    g = res.geom
    # brute force: per block, Eq. (1) on the companded integers, kept range (Eq. (17))
    for br in res.blocks:
        o0, n_out = g.kept(br.w)
        want = brute_conv([int(v) for v in br.s_int], [int(v) for v in res.kernel.k_int])[o0:o0 + n_out]
        assert [int(v) for v in br.r_int] == want
    assert res.out.shape[0] == L + N - 1
    # geometry covers every output once: compare against a per-output recomputation
    full = O.full_precision(s, k)
    assert O.measured_snr_db(full, res.out) > 15.0    # Eq. (19) predicts ~19.9 dB at Q=7


@pytest.mark.parametrize("L,N,W_block", [(1000, 9, 40), (777, 10, 34), (5, 1, 4), (4097, 64, 1024)])
def test_full_precision_overlap_save_vs_brute_force(L, N, W_block):
    rng = np.random.default_rng(L)
    s, k = rng.normal(size=L), rng.normal(size=N)
    res = O.conv_pipeline(s, k, W_block, O.FULL, 0)
    want = np.array(brute_conv(s, k))
    assert np.max(np.abs(res.out - want)) / np.max(np.abs(want)) < 1e-12   # C16


def test_xcorr_definition():
    rng = np.random.default_rng(2)
    x, q = rng.normal(size=300), rng.normal(size=20)
    want = [sum(x[j + n] * q[n] for n in range(20)) for j in range(300 - 20 + 1)]
    got = O.full_precision(x, q, O.XCORR)
    assert np.allclose(got, want, rtol=0, atol=1e-12)
    res = O.conv_pipeline(x, q, 64, O.FULL, 0, mode=O.XCORR)
    assert np.allclose(res.out, want, rtol=0, atol=1e-12)
    c, j = O.xcorr_score(np.array([1.0, 3.0, 3.0, 2.0]))
    assert (c, j) == (3.0, 1)


def test_delta_kernel_and_zero_block():
    rng = np.random.default_rng(4)
    s = rng.uniform(-1, 1, 500)
    s[100:200] = 0.0
    for packing in (O.SYM, O.ASYM2, O.ASYM3):
        res = O.conv_pipeline(s, [1.0], 8, packing, 31, keep_blocks=True)
        for br in res.blocks:                      # delta kernel: r~ = K_q s~
            o0, n = res.geom.kept(br.w)
            assert np.array_equal(br.r_int, 31 * np.convolve(br.s_int, [1.0])[o0:o0 + n])
    s0 = np.zeros(300)
    res = O.conv_pipeline(s0, rng.normal(size=9), 40, O.SYM, 15)
    assert np.all(res.out == 0.0)


def test_saturating_square_wave_plus_rmax():
    """Square wave matched to the kernel signs attains +R_max = S_q ||k~||_1 (reading
    C3) -- POW2 unpacks it exactly; the paper's eps (Eq. (6)) does not (reading C2)."""
    rng = np.random.default_rng(9)
    k = rng.uniform(-1, 1, 9)
    Q = 5
    k_int, _, _ = O.compand(k, Q)
    s = np.tile(np.sign(k_int[::-1]) + 0.0, 20)   # a run reversed-aligned with k
    s[s == 0] = 1.0
    res_p = O.conv_pipeline(s, k, 40, O.SYM, Q, eps_rule=O.EPS_PAPER, rmax_rule=O.RMAX_L1, keep_blocks=True)
    assert max(int(np.max(br.r_exact)) for br in res_p.blocks) == res_p.kernel.R
    assert res_p.mismatches > 0
    res_2 = O.conv_pipeline(s, k, 40, O.SYM, Q, eps_rule=O.EPS_POW2, rmax_rule=O.RMAX_L1)
    assert res_2.mismatches == 0


# --------------------------------------------------------------------------- SNR model pins

def test_eq19_reproduces_paper_166():
    sig = 128.0 / math.sqrt(3.0)                   # uniform [-128, 128]
    for Q, key in ((16, "snr_pred_sym_q16_db"), (256, "snr_pred_asym2_q256_db")):
        got = O.snr_db(sig, sig, 128.0, 128.0, Q, Q)
        assert abs(got - GOLD[key]["value"]) <= GOLD[key]["tol"], got


def test_eq18_closed_form_scaling():
    # doubling S_q and K_q divides the first two D_r terms by 4 and the third by 16
    lin1 = O.snr_linear(1.0, 1.0, 1.0, 1.0, 8, 8)
    lin2 = O.snr_linear(1.0, 1.0, 1.0, 1.0, 16, 16)
    v1 = 1 / (8 * math.sqrt(12))
    v2 = v1 / 2
    assert math.isclose(lin1, 1 / (2 * v1 ** 2 + v1 ** 4), rel_tol=1e-14)
    assert math.isclose(lin2, 1 / (2 * v2 ** 2 + v2 ** 4), rel_tol=1e-14)
    # Table 1's printed cell swaps the pairing (reading C10): differs when peaks/sigmas differ
    s_s, s_k, S, K = 0.2, 0.6, 16, 64
    eq18 = 10 * math.log10(O.snr_linear(s_s, s_k, 1.0, 1.0, S, K))
    printed = 10 * math.log10(144 * (s_s * s_k * S * K) ** 2 / (12 * ((s_s * K) ** 2 + (s_k * S) ** 2) + 1))
    assert abs(eq18 - printed) > 5


@pytest.mark.slow
def test_measured_snr_table2():
    """Table 2: Monte-Carlo of the §IV.A workload (uniform [-128,128], N=800)
    on a 2^18-sample slice, W = 32768: 27.5 dB (S_q=K_q=16) and 51.3 dB (256) +- 1 dB."""
    s, k = WL.paper_iva(seed=0, L=1 << 18)
    Np = 801
    full = O.full_precision(s, k)
    for packing, Q, rmax, key in ((O.SYM, 16, O.RMAX_L1, "snr_meas_sym_q16_db"),
                                  (O.ASYM3, 16, O.RMAX_L1, "snr_meas_asym3_q16_db"),
                                  (O.ASYM2, 256, O.RMAX_L1, "snr_meas_asym2_q256_db")):
        res = O.conv_pipeline(s, k, 32768 + Np + 1, packing, Q, rmax_rule=rmax)
        assert res.kernel.bound_ok and res.mismatches == 0
        got = O.measured_snr_db(full, res.out)
        assert abs(got - GOLD[key]["value"]) <= GOLD[key]["tol"], (key, got)


def test_flop_model_table1():
    f = GOLD["flops_n800"]
    assert O.flop_count(O.FULL, "time", 800) == f["full_time"]
    assert O.flop_count(O.SYM, "time", 800) == f["sym_time"]
    assert O.flop_count(O.ASYM2, "time", 800) == f["asym2_time"]
    # Table 1's ranking: symmetric < asym3 < asym2 < full in time-domain FLOP
    for N in (32, 800, 8192):
        t = [O.flop_count(m, "time", N) for m in (O.SYM, O.ASYM3, O.ASYM2, O.FULL)]
        assert t == sorted(t)


def test_block_sigma():
    assert O.block_sigma([1, -1, 1, -1]) == (1.0, 1.0)
    assert O.block_sigma([0, 0, 0]) == (0.0, 0.0)
    rng = np.random.default_rng(0)
    x = rng.uniform(-128, 128, 1 << 20)
    sig, p = O.block_sigma(x)
    assert abs(sig - 128 / math.sqrt(3)) < 0.2


def test_adapt_spec_example():
    ex = GOLD["adapt_example"]
    kp = np.ones(801)
    assert O.max_q_under_bound(kp, 801, O.SYM, O.EPS_PAPER, O.RMAX_PAPER) == ex["sym_Q"]
    assert O.max_q_under_bound(kp, 801, O.ASYM2, O.EPS_PAPER, O.RMAX_PAPER) == ex["asym2_Q"]
    sig = 128 / math.sqrt(3)
    assert O.snr_db(sig, sig, 128, 128, ex["sym_Q"], ex["sym_Q"]) < ex["floor_db"]
    assert O.snr_db(sig, sig, 128, 128, ex["asym2_Q"], ex["asym2_Q"]) >= ex["floor_db"]
    rng = np.random.default_rng(0)
    s, k = rng.uniform(-128, 128, 20000), rng.uniform(-128, 128, 800)
    dec, qm = O.adapt_decisions(s, k, 3 * 801 + 1, ex["floor_db"], eps_rule=O.EPS_PAPER, rmax_rule=O.RMAX_PAPER)
    assert qm == {O.SYM: 11, O.ASYM2: 232}
    assert all(d[0] == O.ASYM2 for d in dec)
    dec0, _ = O.adapt_decisions(s, k, 3 * 801 + 1, 0.0, eps_rule=O.EPS_PAPER, rmax_rule=O.RMAX_PAPER)
    assert all(d[0] == O.SYM for d in dec0)
    dinf, _ = O.adapt_decisions(s, k, 3 * 801 + 1, math.inf, eps_rule=O.EPS_PAPER, rmax_rule=O.RMAX_PAPER)
    assert all(d[0] == O.FULL for d in dinf)


def test_stereo_workload_delay_and_pairs():
    """NEXT-3 generator: right = left delayed by d (plus 40 dB noise), mono = identical; the
    padded pairs expose all 2B-1 lags and the brute-force xcorr peaks at lag -d."""
    from paper_1201_3018_b200 import workloads as WL
    d = 17
    left, right = WL.stereo(seed=3, seconds=0.2, delay=d)
    noise = right[d:] - left[:-d]
    assert np.sqrt(np.mean(noise ** 2)) < 0.02 * np.sqrt(np.mean(left ** 2))
    l2, r2 = WL.stereo(seed=3, seconds=0.2, delay=0, mono=True)
    assert np.array_equal(l2, r2)
    B = 512
    x, q = WL.stereo_pairs(left, right, B)
    assert x.shape == (len(left) // B, 3 * B - 2) and q.shape == (len(left) // B, B)
    for i in (1, 5):
        c = np.array([np.dot(x[i, j:j + B], q[i]) for j in range(2 * B - 1)])   # valid lags, brute force
        assert int(np.argmax(c)) - (B - 1) == -d


def test_snr_calibration_single_point():
    """P:230 / Fig. 5 (reading C18): the model calibrated by one measurement at S_q = K_q = 8.
    Pins: for the paper's i.i.d. uniform setting Eq. (19)'s assumptions hold, so the
    offset is within 1 dB of zero and the calibrated prediction at Q = 16 lands within 0.5 dB of the
    measurement (P:166 prints 27.1 predicted vs 27.5 measured); at Q = 8 the integer results
    are exact for every packing, so the offset is packing-independent; and model + offset
    reproduces the measurement by construction."""
    rng = np.random.default_rng(11)
    s, k = rng.uniform(-128, 128, 1 << 15), rng.uniform(-128, 128, 401)
    off, meas, model = O.snr_calibration(s, k, 8192, Q=8, packing=O.ASYM2, rmax_rule=O.RMAX_L1)
    assert abs(off) < 1.0 and math.isclose(model + off, meas, rel_tol=0, abs_tol=1e-12)
    for pk in (O.SYM, O.ASYM3):
        off2, meas2, model2 = O.snr_calibration(s, k, 8192, Q=8, packing=pk, rmax_rule=O.RMAX_L1)
        assert meas2 == meas and model2 == model and off2 == off
    out16 = O.conv_pipeline(s, k, 8192, O.ASYM2, 16, rmax_rule=O.RMAX_L1).out
    meas16 = O.measured_snr_db(O.full_precision(s, k), out16)
    _, _, model16 = O.snr_calibration(s, k, 8192, Q=16, packing=O.ASYM2, rmax_rule=O.RMAX_L1)
    assert abs((model16 + off) - meas16) < 0.5
    assert 26.0 < meas16 < 28.5                      # the paper's 27.5 dB regime


def test_validate_backend_u_sys():
    """S:248-256 examples and the guard's purpose: the direct backend compared with itself
    deviates by exactly 0; the FFT backend at N = 3, r_max = 3 stays orders below the paper's
    u_sys (3.1193e-11); its deviation grows with r_max at fixed N; and at N = 801,
    r_max = 51,200 (the §IV.A kernel length) the calibrated u_sys = 4 x deviation is far below
    half the last packed digit (eps = 2^-17 here), so floor-based unpacking stays exact."""
    assert O.validate_backend(801, 51200, trials=5, backend="direct") == (0.0, 0.0)
    d_small, u_small = O.validate_backend(3, 3, trials=100)
    assert d_small < 1e-13 and u_small == 4 * d_small
    d_big, u_big = O.validate_backend(801, 51200, trials=20)
    d_huge, _ = O.validate_backend(801, 12_800_000, trials=20)
    assert d_small < d_big < d_huge
    assert u_big < 0.5 * 2.0 ** -17


# ---------------------------------------------------------------- round 2: L1-rule Q search

def test_max_q_l1_rule_all_ones_801():
    """All-ones 801-tap kernel: k~ = Q * 1 at K_q = Q (Eq. (2), ||k||_inf = 1), so the L1 rule
    R = S_q ||k~||_1 = 801 Q^2 coincides with Eq. (3).  By hand: Table 1's 97,667
    admits 801*11^2 = 96,921 but not 801*12^2 = 115,344 -> Q = 11 (S:401's value); the dyadic
    3-digit bound 131,071 (C4) admits 115,344 but not 801*13^2 = 135,369 -> Q = 12; the dyadic
    2-digit bound 67,108,863 admits 801*289^2 = 66,900,321 but not 801*290^2 = 67,364,100."""
    kp = np.ones(801)
    for rule in (O.RMAX_L1, O.RMAX_PAPER):
        assert O.max_q_under_bound(kp, 801, O.SYM, O.EPS_PAPER, rule) == 11
        assert O.max_q_under_bound(kp, 801, O.SYM, O.EPS_POW2, rule) == 12
        assert O.max_q_under_bound(kp, 801, O.ASYM3, O.EPS_POW2, rule) == 12
        assert O.max_q_under_bound(kp, 801, O.ASYM2, O.EPS_POW2, rule) == 289


def test_max_q_l1_rule_three_tap_hand_example():
    """k = [0.5, -1, 0.25]: c_k = Q, k~ = [[0.5 Q]], -Q, [[0.25 Q]] (round half away, C5).
    L1 rule R(Q) = Q (Q + [[Q/2]] + [[Q/4]]) against the dyadic 3-digit bound 131,071:
      Q = 273: 273 (273 + 137 + 68) = 130,494 <= 131,071
      Q = 274: 274 (274 + 137 + 69) = 131,520 >  131,071   -> Q = 273.
    The PAPER rule R = N' Q^2 = 3 Q^2 gives 3*209^2 = 131,043 <= bound < 3*210^2 = 132,300 -> 209,
    so a search that silently used Eq. (3) instead of the L1 rule fails."""
    kp = np.array([0.5, -1.0, 0.25])
    assert O.max_q_under_bound(kp, 3, O.SYM, O.EPS_POW2, O.RMAX_L1) == 273
    assert O.max_q_under_bound(kp, 3, O.SYM, O.EPS_POW2, O.RMAX_PAPER) == 209
    # the straddling values themselves, by hand
    assert O.companding_range(3, 273, 273, O.compand(kp, 273)[0], O.RMAX_L1) == 130494
    assert O.companding_range(3, 274, 274, O.compand(kp, 274)[0], O.RMAX_L1) == 131520


def test_max_q_l1_rule_scale_invariant_and_monotone():
    """Companding divides by ||k||_inf (Eq. (2)), so scaling k by any power of two leaves
    k~ and hence Q unchanged; a zero tap appended (C13) changes neither ||k~||_1 nor Q."""
    kp = np.array([0.5, -1.0, 0.25])
    for scale in (2.0 ** -7, 1.0, 2.0 ** 9):
        assert O.max_q_under_bound(kp * scale, 3, O.SYM, O.EPS_POW2, O.RMAX_L1) == 273
    assert O.max_q_under_bound(np.append(kp, 0.0), 4, O.SYM, O.EPS_POW2, O.RMAX_L1) == 273


def test_flop_model_frequency_forms_structure():
    """Table 1's frequency-domain FLOP cells are three FFTs of Franchetti's
    5 n log2 n ([13]) at the Table's transform length plus a linear term:
      full  n = 3N+1:      15 n log2 n + n
      sym   same n:        half of full's transform flops + 5N + 1
      asym2 n = 2N+1:      15 n log2 n + 6.5 (3N+1)
      asym3 n = 5N/3+1:    15 n log2 n + (62N + 21) / 3
    A wrong coefficient or transform length in any cell breaks one of these."""
    for N in (3, 32, 800, 8192):
        n_full, n_a2, n_a3 = 3 * N + 1, 2 * N + 1, 5.0 * N / 3.0 + 1
        full = O.flop_count(O.FULL, "freq", N)
        assert math.isclose(full, 15 * n_full * math.log2(n_full) + n_full, rel_tol=1e-12)
        sym = O.flop_count(O.SYM, "freq", N)
        assert math.isclose(sym - (5 * N + 1), 0.5 * (full - n_full), rel_tol=1e-12)
        a2 = O.flop_count(O.ASYM2, "freq", N)
        assert math.isclose(a2, 15 * n_a2 * math.log2(n_a2) + 6.5 * (3 * N + 1), rel_tol=1e-12)
        a3 = O.flop_count(O.ASYM3, "freq", N)
        assert math.isclose(a3, 15 * n_a3 * math.log2(n_a3) + (62 * N + 21) / 3.0, rel_tol=1e-12)
    # "symmetric packing is expected to be the fastest method under both ... domains"
    for N in (32, 800, 8192):
        f = {m: O.flop_count(m, "freq", N) for m in (O.FULL, O.SYM, O.ASYM2, O.ASYM3)}
        assert f[O.SYM] == min(f.values())
