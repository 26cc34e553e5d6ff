"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Plain NumPy float64/int64 oracle of the packed approximate overlap-save convolution of
Anam & Andreopoulos (PAPER.md, cited P:<line>; SPEC.md cited S:<line>).  Each function
follows the paper's equations in the paper's order and notation; library primitives
(np.convolve = direct convolution, Eq. (1)) serve as steps.  No blocking, fusion or
reordering beyond what the paper's overlap-save method states.  Where the paper is
garbled or inconsistent, the reading used is SURVEY.md §8(c)'s, listed in DESIGN.md §3
(codes C1..C17 below refer to those readings).

Pins (tests/test_oracle_*.py, run with -m "not gpu"): brute-force pure-Python
convolution on tiny inputs, the SPEC.md S:300 worked example, exhaustive small sweeps,
Eq. (19)'s 27.1/51.2 dB, Table 2's measured 27.5/51.3 dB, Table 1's
bounds and FLOP forms, invariants.  Functions with no independent pin say
"parity unpinned" in their docstring (none at present).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ----------------------------------------------------------------------------- constants
U_SYS_PAPER = 3.1193e-11            # P:153 "We selected u_sys = 3.1193e-11"
FULL, SYM, ASYM2, ASYM3 = 0, 1, 2, 3
EPS_PAPER, EPS_RADIX, EPS_POW2 = 0, 1, 2
RMAX_PAPER, RMAX_L1 = 0, 1
CONV, XCORR = 0, 1

# Table 1 companding-range bounds, for the paper's epsilon = (2 R_max)^-1.
BOUND_TABLE1 = {SYM: 97667, ASYM3: 97667, ASYM2: 43165096}
# Dyadic epsilon (reading C4): exact iff R(2^{2b}+2^b+1) < 2^53 (3 digits) or
# R(2^b+1) < 2^53 (2 digits), b = ceil(log2(2R+1)).  Derived by pow2_exact() below.


def n_digits(packing: int) -> int:
    """Number of epsilon positions a packed word carries: symmetric uses three
    (eps^0, eps^1, eps^-1, Eq. (9)); asymmetric uses M_asym (Eq. (7))."""
    return {SYM: 3, ASYM2: 2, ASYM3: 3}[packing]


def pow2_exact(R: int, digits: int) -> bool:
    """Reading C4: with eps = 2^-b every packed word, product and partial sum is an
    integer multiple of 2^-b (sym/asym2) or 2^-2b (asym3) of magnitude below
    R * (sum of the digit weights); exact in binary64 iff that count is < 2^53."""
    b = (2 * R).bit_length()
    span = (1 << (2 * b)) + (1 << b) + 1 if digits == 3 else (1 << b) + 1
    return R * span < (1 << 53)


def pow2_bound(packing: int) -> int:
    """Largest R with pow2_exact (131071 for three digits, 67108863 for two)."""
    d = n_digits(packing)
    lo, hi = 1, 1 << 40
    while lo < hi:
        mid = (lo + hi + 1) // 2
        if pow2_exact(mid, d):
            lo = mid
        else:
            hi = mid - 1
    return lo


# ----------------------------------------------------------------------------- rounding

def rhaz(x):
    """[[.]] of Eq. (2): round half away from zero (reading C5).
    Exact for every float64: trunc and the fraction x - trunc(x) are exact."""
    x = np.asarray(x, dtype=np.float64)
    t = np.trunc(x)
    return t + np.sign(x) * (np.abs(x - t) >= 0.5)


# ----------------------------------------------------------------------------- companding

def compand(x, Q):
    """Eq. (2) with uniform companding: c = Q / ||x||_inf, x~ = [[c x]].
    All-zero input: c = 1.  Returns (x~ as float64 integers, c, peak)."""
    x = np.asarray(x, dtype=np.float64)
    peak = float(np.max(np.abs(x))) if x.size else 0.0
    c = 1.0 if peak == 0.0 else float(Q) / peak
    return rhaz(c * x), c, peak


def inverse_compand(r_int, c_s, c_k):
    """Eq. (16): r = (c_s c_k)^-1 r~ -- the inverse (c_s c_k)^-1 is formed once
    per block (one product, one IEEE division) and multiplies every r~ (reading C11)."""
    inv = 1.0 / (c_s * c_k)
    return np.asarray(r_int, dtype=np.float64) * inv


# ----------------------------------------------------------------------------- geometry

@dataclass
class Geometry:
    """Overlap-save geometry (Eq. (10), Eq. (17); reading C7).

    N' = N for odd N, N + 1 for even N (one trailing zero tap, C13).
    W  = W_block - N' - 1   (W_block = W + N + 1), W even, W >= 2N'.
    P  = ceil(L / W) blocks.  Block 0 reads input [0, W_block); block w >= 1 reads
    [wW - 2, wW - 2 + W_block) (implied by Eq. (17) with W_start = (N'-1)/2).
    Kept local outputs: block 0 [0, W + N' - 1); block w >= 1 [N'+1, N'+1+W)
    placed at global N' - 1 + wW + m (Eq. (17)).
    """
    L: int
    N: int
    W_block: int
    Np: int = 0
    W: int = 0
    P: int = 0

    def __post_init__(self):
        self.Np = self.N if self.N % 2 == 1 else self.N + 1
        self.W = self.W_block - self.Np - 1
        if self.L < 1 or self.N < 1:
            raise ValueError("L and N must be >= 1")
        if self.W < 2 or self.W % 2 or self.W < 2 * self.Np:
            raise ValueError(f"W = W_block - N' - 1 = {self.W} must be even and >= 2N' (P:45)")
        self.P = -(-self.L // self.W)

    @property
    def L_out(self):
        return self.L + self.N - 1

    def block_start(self, w):
        return 0 if w == 0 else w * self.W - 2

    def kept(self, w):
        """(first kept local output index, number of kept outputs) of block w."""
        return (0, self.W + self.Np - 1) if w == 0 else (self.Np + 1, self.W)

    def block_input(self, s, w):
        """The W_block samples of block w; samples past L are zero (C7)."""
        g0 = self.block_start(w)
        out = np.zeros(self.W_block, dtype=np.float64)
        seg = s[g0:min(g0 + self.W_block, self.L)]
        out[:seg.shape[0]] = seg
        return out


# ----------------------------------------------------------------------------- R_max, eps

def companding_range(Np, S_q, K_q, k_int=None, rule=RMAX_PAPER):
    """Eq. (3): R_max = [[N S_q K_q]] with N -> N' (C3).  rule=RMAX_L1 gives the
    attainable worst case S_q * ||k~||_1 of r~ = s~ * k~ (C3)."""
    if rule == RMAX_PAPER:
        return int(Np) * int(S_q) * int(K_q)
    return int(S_q) * int(np.sum(np.abs(np.asarray(k_int, dtype=np.int64))))


@dataclass
class Eps:
    eps: float       # packing coefficient epsilon
    eps_inv: float   # 1/epsilon, an exact integer in every rule
    b: int           # log2(eps_inv) for POW2, else 0


def packing_coefficient(R, rule=EPS_POW2):
    """Eq. (6): eps = (2 R_max)^-1 (rule EPS_PAPER).  Reading C2: a radix of
    2R+1 (EPS_RADIX) holds all 2R+1 values of [-R, R]; reading C4: the dyadic
    eps = 2^-b, b = ceil(log2(2R+1)) (EPS_POW2, default)."""
    if rule == EPS_PAPER:
        return Eps(1.0 / (2.0 * R), float(2 * R), 0)
    if rule == EPS_RADIX:
        return Eps(1.0 / (2.0 * R + 1.0), float(2 * R + 1), 0)
    b = (2 * R).bit_length()          # smallest b with 2R + 1 <= 2^b
    return Eps(math.ldexp(1.0, -b), math.ldexp(1.0, b), b)


def bound_for(packing, eps_rule):
    """Table 1 for the paper's / radix epsilon; the exactness bound (C4) for POW2."""
    if eps_rule == EPS_POW2:
        return pow2_bound(packing)
    return BOUND_TABLE1[packing]


# ----------------------------------------------------------------------------- packing

def pack_symmetric_signal(s_int, eps):
    """Eq. (4): s_bar[m] = s~[2m] + eps s~[2m+1], one product then one sum."""
    s_int = np.asarray(s_int, dtype=np.float64)
    if s_int.shape[0] % 2:
        s_int = np.append(s_int, 0.0)
    return s_int[0::2] + eps * s_int[1::2]


def pack_symmetric_kernel(k_int, eps_inv):
    """Eq. (5) with reading C1 (parities swapped so Eqs. (12)-(15) unpack exactly):
    k_bar[n] = k~[2n+1] + eps^-1 k~[2n], n < ceil(N'/2), k~[N'] = 0."""
    k_int = np.asarray(k_int, dtype=np.float64)
    if k_int.shape[0] % 2:
        k_int = np.append(k_int, 0.0)
    return k_int[1::2] + eps_inv * k_int[0::2]


def pack_asymmetric_signal(s_loc, eps, M, o0, S, Np):
    """Eq. (7) with reading C8: segment q covers local outputs [o0+qS, o0+(q+1)S);
    word i (0 <= i < S + N' - 1) packs s_loc[o0 + qS - (N'-1) + i] at eps^q, local
    samples outside [0, W_block) being zero.  Horner, most significant segment last:
    v = s_{M-1}; v = s_q + eps * v for q = M-2 .. 0 (one product, one sum each)."""
    s_loc = np.asarray(s_loc, dtype=np.float64)
    n = S + Np - 1
    segs = []
    for q in range(M):
        idx = o0 + q * S - (Np - 1) + np.arange(n)
        ok = (idx >= 0) & (idx < s_loc.shape[0])
        seg = np.zeros(n)
        seg[ok] = s_loc[idx[ok]]
        segs.append(seg)
    v = segs[M - 1]
    for q in range(M - 2, -1, -1):
        v = segs[q] + eps * v
    return v


# ----------------------------------------------------------------------------- unpacking

def unpack_balanced_sym(rbar, eps_inv):
    """Symmetric three-digit decode (reading C6, balanced digits):
    r_bar = A + eps B + eps^-1 C with |A|,|B|,|C| <= R  (Eq. (9) under C1).
    C = rint(r_bar / eps^-1); rem = r_bar - C eps^-1; A = rint(rem); B = rint((rem-A) eps^-1)."""
    rbar = np.asarray(rbar, dtype=np.float64)
    C = np.rint(rbar / eps_inv)
    rem = rbar - C * eps_inv
    A = np.rint(rem)
    B = np.rint((rem - A) * eps_inv)
    return A, B, C


def assemble_sym(A, B, C, first_is_seed):
    """Eqs. (14)-(15) recombination under C1: r~[2m+1] = A[m] and
    r~[2m] = C[m] + B[m-1] (the one-sample lag of Eq. (12)).  If first_is_seed the
    first packed output is the seeded m = W_start whose even output is discarded
    (footnote 2); otherwise (block 0) B[-1] = 0 (the seed is a true 0)."""
    n = A.shape[0]
    Bprev = np.concatenate([[0.0], B[:-1]])
    r = np.empty(2 * n)
    r[0::2] = C + Bprev
    r[1::2] = A
    return r[2:] if first_is_seed else r


def unpack_paper_sym(rbar, R, eps, eps_inv, u_sys, W_start):
    """Literal Eqs. (11)-(15) on packed outputs m = W_start .. : returns
    (even r~[2m], odd r~[2m+1]) for every m (the seeded even output included).
    Valid only under reading C1 and R < 1/(2 sqrt(u_sys)) (reading C6)."""
    rbar = np.asarray(rbar, dtype=np.float64)
    R_safe = R * (eps + 1.0 + eps_inv) + u_sys * eps_inv
    u = rbar + R_safe                                              # Eq. (11)
    side_eps = np.empty_like(u)
    side_eps[0] = R                                                # Eq. (12), m = W_start
    side_eps[1:] = eps_inv * (u[:-1] - np.floor(u[:-1]))           # Eq. (12), m > W_start
    side_epsinv = np.floor(eps * u)                                # Eq. (13)
    even = np.floor(side_epsinv + side_eps - 2.0 * R)              # Eq. (14)
    odd = np.floor(np.floor(u) - eps_inv * side_epsinv - R)        # Eq. (15)
    return even, odd


def unpack_balanced_asym(rbar, eps_inv, M):
    """Asymmetric decode, "M_asym successive iterations" (procedure of [8] not in
    the paper, reading C9): balanced digits, most significant first:
    t_0 = rint(v); v <- (v - t_0) eps^-1; ... t_{M-1} = rint(v)."""
    v = np.asarray(rbar, dtype=np.float64)
    out = []
    for q in range(M):
        t = np.rint(v)
        out.append(t)
        if q < M - 1:
            v = (v - t) * eps_inv
    return out


def unpack_floor_asym(rbar, R, eps, eps_inv, M, u_sys=0.0):
    """S:330's positive-domain floor iteration (the form SPEC.md derives from [8]):
    u = v + R sum_q eps^q + u_sys; t_q = floor(u) - R, u <- eps^-1 (u - floor(u));
    last t = [[u]] - R.  Exact iff radix >= 2R+1 (reading C2)."""
    u = np.asarray(rbar, dtype=np.float64) + R * sum(eps ** q for q in range(M)) + u_sys
    out = []
    for q in range(M - 1):
        f = np.floor(u)
        out.append(f - R)
        u = eps_inv * (u - f)
    out.append(rhaz(u) - R)
    return out


# ----------------------------------------------------------------------------- kernel state

@dataclass
class KernelState:
    """Initialization step: ||k||_inf, c_k, k~ (Eq. (2)), R_max (Eq. (3)), eps
    (Eq. (6)), packed kernel (Eq. (5)/C1, or k~ for asymmetric, Eq. (8))."""
    k_padded: np.ndarray
    c_k: float
    k_int: np.ndarray
    R: int
    eps: Eps
    packing: int
    bound: int
    bound_ok: bool
    k_packed: np.ndarray = field(default=None)


def prepare_kernel(k, geom: Geometry, packing, S_q, K_q=None, mode=CONV,
                   eps_rule=EPS_POW2, rmax_rule=RMAX_PAPER):
    """Kernel companding once.  xcorr: the kernel is reversed
    before companding (a9).  Even N padded with one trailing zero tap (C13)."""
    K_q = S_q if K_q is None else K_q
    k = np.asarray(k, dtype=np.float64)
    if mode == XCORR:
        k = k[::-1]
    kp = np.zeros(geom.Np)
    kp[:k.shape[0]] = k
    if packing == FULL:
        return KernelState(kp, 1.0, kp, 0, Eps(0.0, 0.0, 0), FULL, 0, True, kp)
    k_int, c_k, _ = compand(kp, K_q)
    R = companding_range(geom.Np, S_q, K_q, k_int, rmax_rule)
    R = max(R, 1)
    e = packing_coefficient(R, eps_rule)
    bound = bound_for(packing, eps_rule)
    st = KernelState(kp, c_k, k_int, R, e, packing, bound, R <= bound)
    st.k_packed = pack_symmetric_kernel(k_int, e.eps_inv) if packing == SYM else k_int
    return st


# ----------------------------------------------------------------------------- per block

@dataclass
class BlockResult:
    w: int
    peak: float
    c_s: float
    s_int: np.ndarray        # W_block companded samples (Eq. (2))
    packed: np.ndarray       # packed words as the conv core sees them (Eq. (4)/(7))
    rbar: np.ndarray         # packed convolution outputs (Eq. (9)/(8))
    r_int: np.ndarray        # unpacked integer outputs of the kept range
    r_exact: np.ndarray      # exact int64 s~ * k~ over the kept range (self-check O9)
    out: np.ndarray          # dequantized kept outputs (Eq. (16))


def process_block(s, w, geom: Geometry, ks: KernelState, S_q, unpack_form="balanced",
                  u_sys=U_SYS_PAPER):
    """One iteration of the per-block loop for block w."""
    blk = geom.block_input(s, w)
    o0, n_out = geom.kept(w)
    Np = geom.Np
    if ks.packing == FULL:
        y = np.convolve(blk, ks.k_padded)                     # Eq. (1), direct
        out = y[o0:o0 + n_out]
        return BlockResult(w, float(np.max(np.abs(blk))), 1.0, blk, blk, y, out, out, out)

    s_int, c_s, peak = compand(blk, S_q)                       # Eq. (2), block companding
    r_exact = np.convolve(s_int.astype(np.int64), ks.k_int.astype(np.int64))[o0:o0 + n_out]
    e = ks.eps
    if ks.packing == SYM:
        K = (Np + 1) // 2
        W_start = 0 if w == 0 else K - 1                       # Eq. (10)
        packed = pack_symmetric_signal(s_int, e.eps)           # Eq. (4), W_block/2 words
        # Eq. (9): r_bar[m] = sum_n s_bar[m-n] k_bar[n], for W_start <= m < W_block/2
        m_hi = (geom.W_block // 2) if w > 0 else (geom.W + Np - 1) // 2
        rbar = np.convolve(packed, ks.k_packed)[W_start:m_hi]
        if unpack_form == "paper":
            even, odd = unpack_paper_sym(rbar, ks.R, e.eps, e.eps_inv, u_sys, W_start)
            r = np.empty(2 * rbar.shape[0])
            r[0::2], r[1::2] = even, odd
            r_int = r[2:] if w > 0 else r     # block 0: the R_max seed encodes B[-1] = 0
        else:
            A, B, C = unpack_balanced_sym(rbar, e.eps_inv)
            r_int = assemble_sym(A, B, C, first_is_seed=(w > 0))
    else:
        M = 2 if ks.packing == ASYM2 else 3
        S = -(-n_out // M)                                     # segment length (C8)
        packed = pack_asymmetric_signal(s_int, e.eps, M, o0, S, Np)   # Eq. (7)
        rbar = np.convolve(packed, ks.k_int, mode="valid")     # Eq. (8), S outputs
        digits = unpack_balanced_asym(rbar, e.eps_inv, M)
        r_int = np.concatenate(digits)[:n_out]
    out = inverse_compand(r_int, c_s, ks.c_k)                  # Eq. (16)
    return BlockResult(w, peak, c_s, s_int, packed, rbar, r_int, r_exact, out)


# ----------------------------------------------------------------------------- pipeline

@dataclass
class PipelineResult:
    out: np.ndarray
    blocks: list
    kernel: KernelState
    geom: Geometry
    mismatches: int


def conv_pipeline(s, k, W_block, packing, Q, K_q=None, mode=CONV, eps_rule=EPS_POW2,
                  rmax_rule=RMAX_PAPER, unpack_form="balanced", u_sys=U_SYS_PAPER,
                  blocks=None, keep_blocks=False):
    """Whole hot path: plan, kernel companding, per block
    companding + packing + packed convolution + unpacking + inverse companding, output
    assembly (Eq. (17)), trimmed to L+N-1 outputs (conv) or to the L-N+1 valid lags
    c[j] = sum_n s[j+n] q[n] (xcorr, reading C17).  ``blocks`` limits the run to a
    subset (for sampled parity at full size); outputs of other blocks are NaN."""
    s = np.asarray(s, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    geom = Geometry(s.shape[0], k.shape[0], W_block)
    ks = prepare_kernel(k, geom, packing, Q, K_q, mode, eps_rule, rmax_rule)
    y = np.full(geom.L_out, np.nan) if blocks is not None else np.zeros(geom.L_out)
    res, mism = [], 0
    for w in (range(geom.P) if blocks is None else blocks):
        br = process_block(s, w, geom, ks, Q, unpack_form, u_sys)
        g0 = geom.block_start(w)
        o0, n_out = geom.kept(w)
        lo = g0 + o0
        n = min(n_out, geom.L_out - lo)
        if n > 0:
            y[lo:lo + n] = br.out[:n]
        if packing != FULL:
            mism += int(np.sum(br.r_int != br.r_exact))
        if keep_blocks:
            res.append(br)
    if mode == XCORR:
        y = y[geom.N - 1:geom.L]                              # valid lags 0 .. L-N
    return PipelineResult(y, res, ks, geom, mism)


def full_precision(s, k, mode=CONV):
    """Eq. (1) single-shot direct FP64 convolution; xcorr = convolution with the
    time-reversed kernel, valid lags only (C17)."""
    s = np.asarray(s, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    if mode == XCORR:
        return np.convolve(s, k[::-1])[k.shape[0] - 1:s.shape[0]]
    return np.convolve(s, k)


def xcorr_score(c):
    """a9 / C17: per-signal max over valid lags and its argmax (lowest lag on ties)."""
    j = int(np.argmax(c))          # numpy returns the first maximal index
    return float(c[j]), j


# ----------------------------------------------------------------------------- SNR model

SQRT12 = math.sqrt(12.0)


def snr_linear(sigma_s, sigma_k, peak_s, peak_k, S_q, K_q):
    """Eqs. (18)-(19) with sigma_v = ||.||_inf / (Q sqrt(12)), as
    the linear ratio N(sigma_s sigma_k)^2 / D_r (N cancels).  Fixed evaluation order:
    this exact sequence of IEEE products and sums is the decision arithmetic (C12).
    (Not Table 1's printed SNR cell, whose S_q/K_q pairing is swapped -- reading C10.)"""
    v_s = peak_s / (S_q * SQRT12)
    v_k = peak_k / (K_q * SQRT12)
    a = sigma_s * v_k
    b = sigma_k * v_s
    c = v_k * v_s
    D = (a * a + b * b) + c * c
    n = sigma_s * sigma_k
    return (n * n) / D


def snr_db(sigma_s, sigma_k, peak_s, peak_k, S_q, K_q, calib_offset_db=0.0):
    """Eq. (19) in dB plus the single-point calibration offset."""
    return 10.0 * math.log10(snr_linear(sigma_s, sigma_k, peak_s, peak_k, S_q, K_q)) + calib_offset_db


def measured_snr_db(ref, approx):
    """10 log10(sum ref^2 / sum (ref-approx)^2); +inf when exact."""
    ref = np.asarray(ref, dtype=np.float64)
    err = float(np.sum((ref - np.asarray(approx, dtype=np.float64)) ** 2))
    return math.inf if err == 0.0 else 10.0 * math.log10(float(np.sum(ref * ref)) / err)


def block_sigma(blk):
    """Marginal sigma of a block ("the square root of its second moment"),
    order-independent (reading C12): z = [[x * (2^20 / p)]] on a fixed integer grid,
    sigma = p * sqrt(sum z^2 / n) / 2^20 with an exact int64 sum.  Returns (sigma, p)."""
    blk = np.asarray(blk, dtype=np.float64)
    p = float(np.max(np.abs(blk)))
    if p == 0.0:
        return 0.0, 0.0
    z = rhaz(blk * (1048576.0 / p)).astype(np.int64)
    m2 = float(np.sum(z * z)) / float(blk.shape[0])
    return p * math.sqrt(m2) / 1048576.0, p


def kernel_sigma(k):
    """sigma_k of the kernel by the same rule as block_sigma."""
    return block_sigma(k)


def max_q_under_bound(k_padded, Np, packing, eps_rule, rmax_rule, q_cap=1 << 15):
    """Largest tied Q = S_q = K_q whose R_max (Eq. (3) or L1) satisfies the mode's bound
    ("selecting the maximum S_q and K_q that allow for this packing").
    R(Q) is nondecreasing in Q under both rules, so a linear scan from the top is exact."""
    bound = bound_for(packing, eps_rule)
    best = 0
    for Q in range(1, q_cap + 1):
        k_int = compand(k_padded, Q)[0] if rmax_rule == RMAX_L1 else None   # Eq. (2) at K_q = Q
        R = companding_range(Np, Q, Q, k_int, rmax_rule)                  # Eq. (3) / C3
        if R <= bound:
            best = Q
        else:
            break
    return best


def snr_threshold_linear(floor_db, calib_offset_db=0.0):
    """The floor as a linear SNR: predicted_db >= floor  <=>  lin >= 10^((floor-off)/10)."""
    return math.pow(10.0, (floor_db - calib_offset_db) / 10.0)


def adapt_decisions(s, k, W_block, floor_db, calib_offset_db=0.0, candidates=(SYM, ASYM2),
                    eps_rule=EPS_POW2, rmax_rule=RMAX_L1, blocks=None):
    """§IV.D adaptation: per block, the first candidate packing (fastest
    first) whose predicted SNR at its maximum Q under its bound meets the floor, else
    full precision (SNR = infinity).  Returns (list of (mode, Q, snr_lin) per block,
    {mode: Q})."""
    s = np.asarray(s, dtype=np.float64)
    geom = Geometry(s.shape[0], len(k), W_block)
    kp = np.zeros(geom.Np)
    kp[:len(k)] = k
    sig_k, pk = kernel_sigma(kp)
    qmode = {m: max_q_under_bound(kp, geom.Np, m, eps_rule, rmax_rule) for m in candidates}
    thr = snr_threshold_linear(floor_db, calib_offset_db)
    out = []
    for w in (range(geom.P) if blocks is None else blocks):
        sig_s, ps = block_sigma(geom.block_input(s, w))
        dec = (FULL, 0, math.inf)
        if sig_s > 0.0:
            for m in candidates:
                Q = qmode[m]
                if Q < 1:
                    continue
                lin = snr_linear(sig_s, sig_k, ps, pk, Q, Q)
                if lin >= thr:
                    dec = (m, Q, lin)
                    break
        else:
            dec = (candidates[0], qmode[candidates[0]], math.inf)  # all-zero block: exact
        out.append(dec)
    return out, qmode


def snr_calibration(s, k, W_block, Q=8, packing=ASYM2, mode=CONV, eps_rule=EPS_POW2, rmax_rule=RMAX_PAPER):
    """Single-point calibration of the Eq. (19) SNR model (Fig. 5: "calibrated via a
    single measurement at the coarsest quantization (S_q = K_q = 8)"; reading C18).  Measure
    the packed pipeline's SNR against full precision at S_q = K_q = Q over the whole signal,
    predict it with Eq. (19) per block -- signal power (sigma_s sigma_k)^2 and noise D_b of
    snr_linear, blocks of equal size, so the signal-level prediction is sum(signal)/sum(noise)
    -- and return (offset_db = measured - model, measured_db, model_db).  The offset is what
    adapt_decisions adds to every prediction."""
    s = np.asarray(s, dtype=np.float64)
    ref = full_precision(s, k, mode=mode)
    out = conv_pipeline(s, k, W_block, packing, Q, mode=mode, eps_rule=eps_rule, rmax_rule=rmax_rule).out
    measured = measured_snr_db(ref, out)
    geom = Geometry(s.shape[0], len(k), W_block)
    kp = np.zeros(geom.Np)
    kp[:len(k)] = k
    sig_k, pk = kernel_sigma(kp)
    num = 0.0
    den = 0.0
    for w in range(geom.P):
        sig_s, ps = block_sigma(geom.block_input(s, w))
        v_s = ps / (Q * SQRT12)                          # snr_linear's terms, same order
        v_k = pk / (Q * SQRT12)
        a = sig_s * v_k
        b = sig_k * v_s
        c = v_k * v_s
        den += (a * a + b * b) + c * c
        n = sig_s * sig_k
        num += n * n
    model = 10.0 * math.log10(num / den)
    return measured - model, measured, model


def validate_backend(N, r_max, trials=100, seed=0, backend="fft"):
    """Backend validation behind the u_sys guard (the paper's u_sys = 3.1193e-11 is
    a machine-precision measurement): convolve `trials` randomized worst-case packed
    operands -- asymmetric M = 2 words of full-magnitude digits +-S_q at the dyadic eps of
    R_max = r_max (Eq. (7) Horner order), kernel digits +-K_q with N S_q K_q ~ r_max -- on the
    backend and on the direct (exact, np.convolve) one, and return (max |deviation|,
    u_sys = 4 max |deviation|) ("measure max fft deviation on integer inputs, scale by
    safety factor 4").  backend: "fft" (NumPy's real FFT, the Tier-2 FFT core of the CPU spec)
    or "direct" (self-comparison: 0)."""
    rng = np.random.default_rng(seed)
    q = max(1, int(math.isqrt(max(1, r_max // max(1, N)))))         # S_q = K_q with N S_q K_q <= r_max
    eps = 1.0 / (1 << (int(2 * r_max).bit_length()))              # reading C4: 2^-b, b = ceil(log2(2R+1))
    n_sig = 4 * N
    dev = 0.0
    for _ in range(trials):
        d0 = q * rng.choice([-1.0, 1.0], n_sig)
        d1 = q * rng.choice([-1.0, 1.0], n_sig)
        x = d0 + eps * d1                                         # Eq. (7), M = 2
        k = q * rng.choice([-1.0, 1.0], N)
        exact = np.convolve(x, k)
        if backend == "direct":
            got = np.convolve(x, k)
        else:
            n = 1 << int(n_sig + N - 1 - 1).bit_length()
            got = np.fft.irfft(np.fft.rfft(x, n) * np.fft.rfft(k, n), n)[:n_sig + N - 1]
        dev = max(dev, float(np.max(np.abs(got - exact))))
    return dev, 4.0 * dev


# ----------------------------------------------------------------------------- Table 1

def flop_count(packing, domain, N):
    """Table 1 FLOP row, verbatim closed forms."""
    if domain == "time":
        return {FULL: 4 * N * N, SYM: N * N + N, ASYM2: 2.5 * N * N - N,
                ASYM3: 2 * N * N - 2.0 / 3.0 * N}[packing]
    lg = math.log2
    return {FULL: (45 * N + 15) * lg(3 * N + 1) + 3 * N + 1,
            SYM: (22.5 * N + 7.5) * lg(3 * N + 1) + 5 * N + 1,
            ASYM2: (30 * N + 15) * lg(2 * N + 1) + 19.5 * N + 6.5,
            ASYM3: (25 * N + 15) * lg(5.0 / 3.0 * N + 1) + 62.0 / 3.0 * N + 7}[packing]


def adaptive_pipeline(s, k, W_block, floor_db, calib_offset_db=0.0, candidates=(SYM, ASYM2),
                      eps_rule=EPS_POW2, rmax_rule=RMAX_L1):
    """§IV.D end to end: per-block decisions (adapt_decisions), then each
    block runs the per-block loop with its chosen packing at that packing's Q (kernel
    companded once per packing).  Returns (output, decisions, qmode)."""
    s = np.asarray(s, dtype=np.float64)
    dec, qmode = adapt_decisions(s, k, W_block, floor_db, calib_offset_db, candidates, eps_rule, rmax_rule)
    geom = Geometry(s.shape[0], len(k), W_block)
    states = {m: prepare_kernel(k, geom, m, qmode[m], None, CONV, eps_rule, rmax_rule)
              for m in candidates if qmode[m] >= 1}
    states[FULL] = prepare_kernel(k, geom, FULL, 0)
    y = np.zeros(geom.L_out)
    for w, (m, Q, _) in enumerate(dec):
        br = process_block(s, w, geom, states[m], Q)
        g0 = geom.block_start(w)
        o0, n_out = geom.kept(w)
        n = min(n_out, geom.L_out - (g0 + o0))
        if n > 0:
            y[g0 + o0:g0 + o0 + n] = br.out[:n]
    return y, dec, qmode
