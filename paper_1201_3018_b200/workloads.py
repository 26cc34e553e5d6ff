"""Seeded synthetic inputs for the BASELINE.json configs (SURVEY.md §8(d) "Synthetic inputs").

This module holds NO arithmetic of the method (no companding, packing, convolution,
unpacking or SNR model) -- only input recipes.  It is the one module shared by the
CPU oracle tests, the GPU parity tests and bench.py (task rule ③).  Every generator
is a pure function of its seed: numpy ``default_rng(seed)`` (PCG64), draws taken in
the order written here (signal first, then kernel).

The paper's own application data (cover-song beat/chroma features [3], MPEG-7 clips
[15]) is not available; these recipes stand in for it.
Where BASELINE.json leaves a detail open the assumption is listed in DESIGN.md §3.
"""
from __future__ import annotations

import numpy as np

FS = 44100.0  # audio sample rate of configs 2 and 4 (BASELINE.json configs[1], [3])

CONFIGS = {
    # name: (L, N, W_block)  -- BASELINE.json configs[0..4]
    "cfg1": (65536, 64, 1024),
    "cfg2": (1 << 22, 512, 4096),
    "cfg3": (1 << 24, 4096, 16384),
    "cfg4": (1 << 20, 8192, 32768),  # per database signal; W_block chosen
    "cfg5": (1 << 26, 1024, 4096),
}


def laplace_clipped(rng: np.random.Generator, n: int, scale: float) -> np.ndarray:
    """i.i.d. Laplace(0, scale) clipped to [-1, 1] (configs 1 and 3)."""
    return np.clip(rng.laplace(0.0, scale, n), -1.0, 1.0)


def sinusoid_mixture(rng: np.random.Generator, n: int, n_sines: int = 16,
                     fmin: float = 50.0, fmax: float = 8000.0, fs: float = FS,
                     block: int = 1024) -> np.ndarray:
    """Sum of ``n_sines`` sinusoids, f log-uniform in [fmin, fmax] Hz, amplitude
    U[0.1, 1], phase U[0, 2pi).  Evaluated per ``block`` samples with the
    angle-addition identity (a small matrix product) so that 2^20..2^26-sample
    signals generate in well under a second."""
    f = np.exp(rng.uniform(np.log(fmin), np.log(fmax), n_sines))
    a = rng.uniform(0.1, 1.0, n_sines)
    ph = rng.uniform(0.0, 2.0 * np.pi, n_sines)
    w = 2.0 * np.pi * f / fs
    nb = -(-n // block)
    t0 = np.arange(nb, dtype=np.float64)[:, None] * block          # block starts
    tau = np.arange(block, dtype=np.float64)[None, :]
    # sin(w(t0+tau)+ph) = sin(w t0 + ph) cos(w tau) + cos(w t0 + ph) sin(w tau)
    ang0 = t0 * w[None, :] + ph[None, :]                             # nb x n_sines
    lhs = np.concatenate([np.sin(ang0) * a, np.cos(ang0) * a], axis=1)
    rhs = np.concatenate([np.cos(w[:, None] * tau), np.sin(w[:, None] * tau)], axis=0)
    return (lhs @ rhs).reshape(-1)[:n]


def add_white_noise(rng: np.random.Generator, x: np.ndarray, snr_db: float) -> np.ndarray:
    p = float(np.mean(x * x)) / (10.0 ** (snr_db / 10.0))
    return x + rng.normal(0.0, np.sqrt(p), x.shape[0])


def pink_noise(rng: np.random.Generator, n: int) -> np.ndarray:
    """1/f-power Gaussian noise: white Gaussian shaped by 1/sqrt(f) in the DFT domain."""
    X = np.fft.rfft(rng.normal(0.0, 1.0, n))
    f = np.arange(X.shape[0], dtype=np.float64)
    X[0] = 0.0
    X[1:] /= np.sqrt(f[1:])
    return np.fft.irfft(X, n)


def normalize_peak(x: np.ndarray) -> np.ndarray:
    return x / np.max(np.abs(x))


def windowed_sinc(N: int, fc: float = 8000.0, fs: float = FS) -> np.ndarray:
    """Blackman-windowed sinc low-pass FIR, cutoff fc (config 2's kernel; window and
    cutoff are not fixed by BASELINE.json -- assumption listed in DESIGN.md)."""
    n = np.arange(N, dtype=np.float64) - (N - 1) / 2.0
    return (2.0 * fc / fs) * np.sinc(2.0 * fc / fs * n) * np.blackman(N)


# ---------------------------------------------------------------------------- configs

def cfg1(seed: int = 0, L: int = 65536, N: int = 64):
    """Config 1: Laplace(0, 0.1) clipped, kernel U[-1, 1]."""
    rng = np.random.default_rng(seed)
    s = laplace_clipped(rng, L, 0.1)
    k = rng.uniform(-1.0, 1.0, N)
    return s, k


def cfg2(seed: int = 0, L: int = 1 << 22, N: int = 512):
    """Config 2: 16-sinusoid audio mixture + Gaussian noise at 30 dB SNR, peak-normalized;
    Blackman-windowed sinc kernel (8 kHz cutoff)."""
    rng = np.random.default_rng(seed)
    s = normalize_peak(add_white_noise(rng, sinusoid_mixture(rng, L), 30.0))
    k = windowed_sinc(N)
    return s, k


def cfg3(seed: int = 0, L: int = 1 << 24, N: int = 4096):
    """Config 3: Laplace(0, 0.2) clipped; kernel i.i.d. N(0, 1/N)."""
    rng = np.random.default_rng(seed)
    s = laplace_clipped(rng, L, 0.2)
    k = rng.normal(0.0, np.sqrt(1.0 / N), N)
    return s, k


def cfg4_signal(i: int, L: int = 1 << 20) -> np.ndarray:
    """Config 4 database signal i (own seed 1000+i so any subset regenerates alone):
    16-sinusoid mixture at 60 dB white-noise SNR plus pink noise at 0.1x its std,
    peak-normalized."""
    rng = np.random.default_rng(1000 + i)
    x = add_white_noise(rng, sinusoid_mixture(rng, L), 60.0)
    p = pink_noise(rng, L)
    x = x + p * (0.1 * np.std(x) / np.std(p))
    return normalize_peak(x)


def cfg4_query(seed: int = 0, n_signals: int = 1024, L: int = 1 << 20, N: int = 8192):
    """Config 4 query: N samples cut at a random offset of a random database signal,
    plus white noise at 20 dB SNR.  Returns (query, signal_index, offset)."""
    rng = np.random.default_rng(seed)
    i0 = int(rng.integers(n_signals))
    off = int(rng.integers(0, L - N))
    q = add_white_noise(rng, cfg4_signal(i0, L)[off:off + N].copy(), 20.0)
    return q, i0, off


def cfg5(seed: int = 0, L: int = 1 << 26, N: int = 1024, gen_block: int = 4096):
    """Config 5: Laplace samples whose scale is log-uniform in [0.01, 1] per 4096-sample
    generator block (not clipped); kernel i.i.d. N(0, 1/N)."""
    rng = np.random.default_rng(seed)
    nb = -(-L // gen_block)
    scales = np.exp(rng.uniform(np.log(0.01), np.log(1.0), nb))
    s = rng.laplace(0.0, 1.0, L) * np.repeat(scales, gen_block)[:L]
    k = rng.normal(0.0, np.sqrt(1.0 / N), N)
    return s, k


def paper_iva(seed: int = 0, L: int = 8192 * 1024, N: int = 800):
    """§IV.A synthetic workload: input and kernel i.i.d. uniform [-128, 128]."""
    rng = np.random.default_rng(seed)
    s = rng.uniform(-128.0, 128.0, L)
    k = rng.uniform(-128.0, 128.0, N)
    return s, k


def uniform_ints(seed: int, n: int, q: int) -> np.ndarray:
    """Integer-valued float64 samples uniform in {-q..q} (integer-domain tests)."""
    rng = np.random.default_rng(seed)
    return rng.integers(-q, q + 1, n).astype(np.float64)


GENERATORS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg5": cfg5}


def stereo(seed: int = 0, seconds: float = 10.0, delay: int = 17, snr_db: float = 40.0, mono: bool = False,
           fs: float = FS):
    """NEXT-3 stand-in for §IV.C's MPEG-7 clips (the clips are not available): a
    synthetic stereo pair.  left = 16-sinusoid mixture + pink noise (0.1x std), peak-normalized;
    right = left delayed by `delay` samples (right[n] = left[n - delay]) plus white noise at
    `snr_db`; mono: right = left exactly.  Returns (left, right)."""
    rng = np.random.default_rng(seed)
    n = int(seconds * fs)
    x = sinusoid_mixture(rng, n + abs(delay))
    p = pink_noise(rng, n + abs(delay))
    x = normalize_peak(x + p * (0.1 * np.std(x) / np.std(p)))
    left = x[abs(delay):abs(delay) + n] if delay >= 0 else x[:n]
    if mono:
        return left.copy(), left.copy()
    right = x[abs(delay) - delay:abs(delay) - delay + n]
    return left, add_white_noise(rng, right, snr_db)


def stereo_pairs(left: np.ndarray, right: np.ndarray, B: int):
    """Blocks b of B samples: x_b = left block with B-1 zeros on each side (so the valid lags
    j = 0..2B-2 of the xcorr are all 2B-1 lags l = j - (B-1)), q_b = right block.  Returns
    (x: n x (3B-2), q: n x B) for the n = len // B whole blocks."""
    n = min(len(left), len(right)) // B
    x = np.zeros((n, 3 * B - 2))
    x[:, B - 1:2 * B - 1] = left[:n * B].reshape(n, B)
    q = right[:n * B].reshape(n, B).copy()
    return x, q
