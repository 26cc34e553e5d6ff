"""Thin ctypes binding of include/packedconv.h (argument marshalling only).

Every function here has the name of the C entry point it wraps (without the ``conv_``
prefix where noted) and does nothing but convert arguments: torch tensors / numpy arrays
-> raw pointers, streams -> cudaStream_t, status codes -> exceptions.  All numeric work
runs in the CUDA kernels of ``libpackedconv.so``.  There is no CPU fallback: if the
library is missing, ``load()`` raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PC_LIB_PATH") or os.path.join(_HERE, "libpackedconv.so")   # override: experiments

PC_OK, PC_E_CONFIG, PC_E_BOUND, PC_E_BACKEND, PC_E_CUDA, PC_W_UNPACK_MARGIN, PC_E_STATE = 0, 2, 3, 4, 5, 6, 7
MODE_CONV, MODE_XCORR = 0, 1
PACK_FULL, PACK_SYM, PACK_ASYM2, PACK_ASYM3, PACK_ADAPTIVE = 0, 1, 2, 3, 4
EPS_PAPER, EPS_RADIX, EPS_POW2 = 0, 1, 2
RMAX_PAPER, RMAX_L1 = 0, 1
BOUND_STRICT, BOUND_WARN = 0, 1
CORE_DIRECT, CORE_FFT = 0, 1
EXEC_FUSED, EXEC_PERBLOCK, EXEC_TILED = 0, 1, 2

PACK_NAMES = {PACK_FULL: "full", PACK_SYM: "sym", PACK_ASYM2: "asym2", PACK_ASYM3: "asym3",
              PACK_ADAPTIVE: "adaptive"}


class conv_opts(C.Structure):
    _fields_ = [("eps_rule", C.c_int32), ("rmax_rule", C.c_int32), ("bound_policy", C.c_int32),
                ("core", C.c_int32), ("exec", C.c_int32), ("K_q", C.c_int32), ("device", C.c_int32),
                ("reserved", C.c_int32 * 9), ("u_sys", C.c_double)]


class conv_plan_info(C.Structure):
    _fields_ = [("L", C.c_int64), ("L_out", C.c_int64), ("P", C.c_int64),
                ("N", C.c_int32), ("Np", C.c_int32), ("W_block", C.c_int32), ("W", C.c_int32),
                ("mode", C.c_int32), ("packing", C.c_int32), ("Q", C.c_int32), ("K_q", C.c_int32),
                ("taps", C.c_int32), ("kernel_set", C.c_int32),
                ("R_max", C.c_int64), ("bound", C.c_int64), ("bound_ok", C.c_int32), ("eps_b", C.c_int32),
                ("eps", C.c_double), ("eps_inv", C.c_double), ("c_k", C.c_double), ("k_peak", C.c_double),
                ("packed_stride", C.c_int64), ("rbar_stride", C.c_int64), ("rint_stride", C.c_int64),
                ("q_mode", C.c_int32 * 4), ("core_tile", C.c_int32), ("fft_n", C.c_int32),
                ("core_mma", C.c_int32)]


class conv_shard(C.Structure):
    _fields_ = [("block_begin", C.c_int64), ("block_end", C.c_int64), ("in_begin", C.c_int64),
                ("in_end", C.c_int64), ("out_begin", C.c_int64), ("out_end", C.c_int64)]


class conv_block_decision(C.Structure):
    _fields_ = [("packing", C.c_int32), ("Q", C.c_int32), ("snr_lin", C.c_double)]


class PcError(RuntimeError):
    def __init__(self, code, where):
        self.code = code
        super().__init__(f"{where}: {status_string(code)} ({code})")


_lib = None


def load():
    """Load the in-tree library (built by __graft_entry__.build()); raises if missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = C.CDLL(LIB_PATH)
        P, I64, I32, D, VP = C.c_void_p, C.c_int64, C.c_int32, C.c_double, C.c_void_p
        sig = {
            "conv_opts_default": (None, [C.POINTER(conv_opts)]),
            "conv_plan_create": (C.c_int, [C.POINTER(P), I64, I32, I32, I32, I32, I32, C.POINTER(conv_opts)]),
            "conv_plan_set_kernel": (C.c_int, [P, VP, VP]),
            "conv_execute": (C.c_int, [P, VP, VP, VP]),
            "conv_execute_blocks": (C.c_int, [P, VP, I64, VP, I64, I64, I64, VP]),
            "conv_execute_batch": (C.c_int, [P, VP, I64, I64, VP, I64, VP]),
            "conv_execute_host": (C.c_int, [P, VP, VP, VP]),
            "conv_xcorr_max": (C.c_int, [P, VP, I64, I64, VP, VP, VP]),
            "conv_plan_set_kernels": (C.c_int, [P, VP, I64, I64, VP]),
            "conv_xcorr_pairs": (C.c_int, [P, VP, I64, I64, VP, VP, VP]),
            "conv_execute_debug": (C.c_int, [P, VP, VP, VP, VP, VP, VP, VP]),
            "conv_adapt_block": (C.c_int, [P, VP, D, D, C.POINTER(conv_block_decision), VP]),
            "conv_snr_calibrate": (C.c_int, [P, VP, VP, I32, C.POINTER(D), C.POINTER(D), C.POINTER(D), VP]),
            "conv_plan_query": (C.c_int, [P, C.POINTER(conv_plan_info)]),
            "conv_execute_profile": (C.c_int, [P, VP, VP, VP, C.POINTER(C.c_int32), VP]),
            "conv_shard_range": (C.c_int, [I64, I32, I32, I32, I32, I32, C.POINTER(conv_shard)]),
            "conv_plan_residual": (C.c_int, [P, C.POINTER(C.c_double), I32, VP]),
            "conv_plan_destroy": (None, [P]),
            "conv_status_string": (C.c_char_p, [C.c_int]),
        }
        for name, (res, args) in sig.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
    return _lib


def _ptr(x):
    """Raw pointer of a torch tensor / numpy array / int / None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if hasattr(x, "ctypes"):
        return x.ctypes.data
    raise TypeError(type(x))


def _stream(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except ImportError:
            pass
        return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _check(rc, where):
    if rc != PC_OK:
        raise PcError(rc, where)


def status_string(code):
    return load().conv_status_string(int(code)).decode()


def opts_default(**kw):
    o = conv_opts()
    load().conv_opts_default(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def plan_create(L, N, W_block, mode=MODE_CONV, packing=PACK_SYM, Q=127, opts=None, **kw):
    o = opts if opts is not None else opts_default(**kw)
    h = C.c_void_p()
    _check(load().conv_plan_create(C.byref(h), int(L), int(N), int(W_block), int(mode), int(packing), int(Q),
                                   C.byref(o)), "conv_plan_create")
    return h


def plan_set_kernel(plan, k_dev, stream=None):
    _check(load().conv_plan_set_kernel(plan, _ptr(k_dev), _stream(stream)), "conv_plan_set_kernel")


def execute(plan, s_dev, r_dev, stream=None):
    _check(load().conv_execute(plan, _ptr(s_dev), _ptr(r_dev), _stream(stream)), "conv_execute")


def execute_blocks(plan, s_dev, s_offset, r_dev, r_offset, block_begin, block_end, stream=None):
    _check(load().conv_execute_blocks(plan, _ptr(s_dev), int(s_offset), _ptr(r_dev), int(r_offset),
                                      int(block_begin), int(block_end), _stream(stream)), "conv_execute_blocks")


def execute_batch(plan, s_dev, n_signals, s_stride, r_dev, r_stride, stream=None):
    _check(load().conv_execute_batch(plan, _ptr(s_dev), int(n_signals), int(s_stride), _ptr(r_dev),
                                     int(r_stride), _stream(stream)), "conv_execute_batch")


def execute_host(plan, s_host, r_host, stream=None):
    _check(load().conv_execute_host(plan, _ptr(s_host), _ptr(r_host), _stream(stream)), "conv_execute_host")


def xcorr_max(plan, db_dev, n_signals, s_stride, score_dev, lag_dev, stream=None):
    _check(load().conv_xcorr_max(plan, _ptr(db_dev), int(n_signals), int(s_stride), _ptr(score_dev),
                                 _ptr(lag_dev), _stream(stream)), "conv_xcorr_max")


def set_kernels(plan, q_dev, n, q_stride, stream=None):
    """One kernel per pair (NEXT-3): n rows of N doubles, row stride q_stride (device)."""
    _check(load().conv_plan_set_kernels(plan, _ptr(q_dev), int(n), int(q_stride), _stream(stream)),
           "conv_plan_set_kernels")


def xcorr_pairs(plan, x_dev, n, x_stride, score_dev, lag_dev, stream=None):
    """score/lag of pair i = (row i of x, kernel i); see include/packedconv.h."""
    _check(load().conv_xcorr_pairs(plan, _ptr(x_dev), int(n), int(x_stride), _ptr(score_dev), _ptr(lag_dev),
                                   _stream(stream)), "conv_xcorr_pairs")


def execute_debug(plan, s_dev, r_dev=None, packed=None, rbar=None, rint=None, c_s=None, stream=None):
    _check(load().conv_execute_debug(plan, _ptr(s_dev), _ptr(r_dev), _ptr(packed), _ptr(rbar), _ptr(rint),
                                     _ptr(c_s), _stream(stream)), "conv_execute_debug")


def adapt_block(plan, s_dev, snr_floor_db, calib_offset_db=0.0, P=None, stream=None):
    """Returns a list of (packing, Q, snr_lin) per block if P is given."""
    out = (conv_block_decision * int(P))() if P else None
    _check(load().conv_adapt_block(plan, _ptr(s_dev), float(snr_floor_db), float(calib_offset_db), out,
                                   _stream(stream)), "conv_adapt_block")
    return [(d.packing, d.Q, d.snr_lin) for d in out] if out is not None else None


def snr_calibrate(plan, s_dev, k_dev, Q=8, stream=None):
    """Single-point SNR-model calibration: returns (offset_db, measured_db, model_db)."""
    off, meas, model = C.c_double(), C.c_double(), C.c_double()
    _check(load().conv_snr_calibrate(plan, _ptr(s_dev), _ptr(k_dev), int(Q), C.byref(off), C.byref(meas),
                                     C.byref(model), _stream(stream)), "conv_snr_calibrate")
    return off.value, meas.value, model.value


def execute_profile(plan, s_dev, r_dev, records_dev, stream=None):
    """Returns the persistent grid size; records_dev (uint64, 4*148*32) gets per-CTA
    {smid, t_start_ns, t_end_ns, blocks}."""
    g = C.c_int32()
    _check(load().conv_execute_profile(plan, _ptr(s_dev), _ptr(r_dev), _ptr(records_dev), C.byref(g),
                                       _stream(stream)), "conv_execute_profile")
    return g.value


def shard_range(L, N, W_block, mode, rank, world):
    """Host-only block-range shard of `rank` (conv_shard_range) as a dict."""
    sh = conv_shard()
    _check(load().conv_shard_range(int(L), int(N), int(W_block), int(mode), int(rank), int(world), C.byref(sh)),
           "conv_shard_range")
    return {name: getattr(sh, name) for name, _ in conv_shard._fields_}


def plan_residual(plan, reset=True, stream=None):
    """FFT core: largest last-digit residual (LSB) since the last reset and the status
    (PC_OK or PC_W_UNPACK_MARGIN if > 0.25 LSB)."""
    r = C.c_double()
    rc = load().conv_plan_residual(plan, C.byref(r), int(bool(reset)), _stream(stream))
    if rc not in (PC_OK, PC_W_UNPACK_MARGIN):
        _check(rc, "conv_plan_residual")
    return r.value, rc


def plan_query(plan):
    info = conv_plan_info()
    _check(load().conv_plan_query(plan, C.byref(info)), "conv_plan_query")
    d = {name: getattr(info, name) for name, _ in conv_plan_info._fields_}
    d["q_mode"] = list(info.q_mode)
    return d


def plan_destroy(plan):
    if plan:
        load().conv_plan_destroy(plan)


class Plan:
    """Owning wrapper: ``with Plan(L, N, W_block, ...) as p: p.set_kernel(k); p.execute(s, r)``."""

    def __init__(self, L, N, W_block, mode=MODE_CONV, packing=PACK_SYM, Q=127, **opts):
        self.h = None
        self.h = plan_create(L, N, W_block, mode, packing, Q, **opts)

    def set_kernel(self, k_dev, stream=None):
        plan_set_kernel(self.h, k_dev, stream)
        return self

    def execute(self, s_dev, r_dev, stream=None):
        execute(self.h, s_dev, r_dev, stream)

    def execute_blocks(self, *a, **k):
        execute_blocks(self.h, *a, **k)

    def execute_batch(self, *a, **k):
        execute_batch(self.h, *a, **k)

    def execute_host(self, *a, **k):
        execute_host(self.h, *a, **k)

    def execute_debug(self, *a, **k):
        execute_debug(self.h, *a, **k)

    def xcorr_max(self, *a, **k):
        xcorr_max(self.h, *a, **k)

    def set_kernels(self, *a, **k):
        set_kernels(self.h, *a, **k)

    def xcorr_pairs(self, *a, **k):
        xcorr_pairs(self.h, *a, **k)

    def adapt_block(self, s_dev, floor_db, calib_offset_db=0.0, stream=None):
        return adapt_block(self.h, s_dev, floor_db, calib_offset_db, self.info()["P"], stream)

    def snr_calibrate(self, s_dev, k_dev, Q=8, stream=None):
        return snr_calibrate(self.h, s_dev, k_dev, Q, stream)

    def info(self):
        return plan_query(self.h)

    def residual(self, reset=True, stream=None):
        return plan_residual(self.h, reset, stream)

    def close(self):
        if getattr(self, "h", None):
            plan_destroy(self.h)
            self.h = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
