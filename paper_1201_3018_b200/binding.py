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

PC_OK, PC_E_CONFIG, PC_E_BOUND, PC_E_BACKEND, PC_E_CUDA, PC_W_UNPACK_MARGIN, PC_E_STATE, PC_E_WATCHDOG = \
    0, 2, 3, 4, 5, 6, 7, 8
MODE_CONV, MODE_XCORR = 0, 1
PACK_FULL, PACK_SYM, PACK_ASYM2, PACK_ASYM3, PACK_ADAPTIVE = 0, 1, 2, 3, 4
EPS_PAPER, EPS_RADIX, EPS_POW2 = 0, 1, 2
RMAX_PAPER, RMAX_L1 = 0, 1
BOUND_STRICT, BOUND_WARN = 0, 1
CORE_DIRECT, CORE_FFT = 0, 1
EXEC_FUSED, EXEC_PERBLOCK, EXEC_TILED = 0, 1, 2
CORE_AUTO, CORE_FMA, CORE_DMMA = 0, 1, 2
UNPACK_BALANCED, UNPACK_LITERAL = 0, 1

PACK_NAMES = {PACK_FULL: "full", PACK_SYM: "sym", PACK_ASYM2: "asym2", PACK_ASYM3: "asym3",
              PACK_ADAPTIVE: "adaptive"}


class conv_opts(C.Structure):
    _fields_ = [("eps_rule", C.c_int32), ("rmax_rule", C.c_int32), ("bound_policy", C.c_int32),
                ("core", C.c_int32), ("exec", C.c_int32), ("K_q", C.c_int32), ("device", C.c_int32),
                ("raw_staging", C.c_int32), ("core_tile", C.c_int32), ("core_variant", C.c_int32),
                ("parts_per_job", C.c_int32), ("fft_n", C.c_int32), ("unpack_form", C.c_int32),
                ("pack_alu", C.c_int32), ("stage_cap", C.c_int32), ("prepack", C.c_int32),
                ("early_fill", C.c_int32), ("validate_trials", C.c_int32), ("u_sys", C.c_double)]


class conv_plan_info(C.Structure):
    _fields_ = [("L", C.c_int64), ("L_out", C.c_int64), ("P", C.c_int64),
                ("N", C.c_int32), ("Np", C.c_int32), ("W_block", C.c_int32), ("W", C.c_int32),
                ("mode", C.c_int32), ("packing", C.c_int32), ("Q", C.c_int32), ("K_q", C.c_int32),
                ("taps", C.c_int32), ("kernel_set", C.c_int32),
                ("R_max", C.c_int64), ("bound", C.c_int64), ("bound_ok", C.c_int32), ("eps_b", C.c_int32),
                ("eps", C.c_double), ("eps_inv", C.c_double), ("c_k", C.c_double), ("k_peak", C.c_double),
                ("packed_stride", C.c_int64), ("rbar_stride", C.c_int64), ("rint_stride", C.c_int64),
                ("q_mode", C.c_int32 * 4), ("core_tile", C.c_int32), ("fft_n", C.c_int32),
                ("core_mma", C.c_int32), ("backend_ok", C.c_int32), ("backend_resid", C.c_double),
                ("u_sys_cal", C.c_double), ("device", C.c_int32), ("exec_used", C.c_int32)]


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
            "conv_execute_host_blocks": (C.c_int, [P, VP, I64, VP, I64, I64, I64, VP]),
            "conv_best_match": (C.c_int, [VP, VP, VP, I64, I64, VP, VP]),
            "conv_xcorr_max": (C.c_int, [P, VP, I64, I64, VP, VP, VP]),
            "conv_plan_set_kernels": (C.c_int, [P, VP, I64, I64, VP]),
            "conv_xcorr_pairs": (C.c_int, [P, VP, I64, I64, VP, VP, VP]),
            "conv_execute_debug": (C.c_int, [P, VP, VP, VP, VP, VP, VP, C.POINTER(C.c_double), VP]),
            "conv_adapt_block": (C.c_int, [P, VP, D, D, C.POINTER(conv_block_decision), VP]),
            "conv_adapt_blocks": (C.c_int, [P, VP, I64, I64, I64, D, D, C.POINTER(conv_block_decision), VP]),
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


def _bad(where, msg):
    raise PcError(PC_E_CONFIG, f"{where}: {msg}")


def _dev(x, n, where, name, info, dtype="float64", optional=False):
    """Pointer of a device buffer the C ABI will read or write `n` elements of: a contiguous
    CUDA tensor of `dtype` on the plan's device with at least n elements (the ABI takes no
    lengths, so a short / strided / wrong-typed / host buffer would be an out-of-bounds access).
    A raw int is passed through unchecked (caller-managed memory)."""
    if x is None:
        if optional:
            return None
        _bad(where, f"{name} is required")
    if isinstance(x, int):
        return x
    if not hasattr(x, "is_cuda") or not x.is_cuda:
        _bad(where, f"{name} must be a CUDA tensor")
    if str(x.dtype) != "torch." + dtype:
        _bad(where, f"{name} must be {dtype}, got {x.dtype}")
    if not x.is_contiguous():
        _bad(where, f"{name} must be contiguous")
    if x.device.index != info["device"]:
        _bad(where, f"{name} is on cuda:{x.device.index}, the plan on cuda:{info['device']}")
    if x.numel() < n:
        _bad(where, f"{name} has {x.numel()} elements, needs {n}")
    return x.data_ptr()


def _host(x, n, where, name):
    """Pointer of a host float64 buffer of at least n elements (numpy array or CPU tensor)."""
    if isinstance(x, int):
        return x
    if hasattr(x, "is_cuda"):
        if x.is_cuda or str(x.dtype) != "torch.float64" or not x.is_contiguous():
            _bad(where, f"{name} must be a contiguous float64 CPU tensor")
        if x.numel() < n:
            _bad(where, f"{name} has {x.numel()} elements, needs {n}")
        return x.data_ptr()
    if hasattr(x, "ctypes"):
        if x.dtype.name != "float64" or not x.flags["C_CONTIGUOUS"]:
            _bad(where, f"{name} must be a C-contiguous float64 array")
        if x.size < n:
            _bad(where, f"{name} has {x.size} elements, needs {n}")
        return x.ctypes.data
    raise TypeError(type(x))


def _rows(n, stride, length):
    """Elements spanned by n rows of `length` at row stride `stride`."""
    return 0 if n <= 0 else (n - 1) * stride + length


def _block_span(info, b0, b1):
    """(input end, output end), global indices, of blocks [b0, b1) (reading C7, Eq. (17))."""
    if b1 <= b0:
        return 0, 0
    L, N, Np, W, Wb = info["L"], info["N"], info["Np"], info["W"], info["W_block"]
    g_last = 0 if b1 - 1 == 0 else (b1 - 1) * W - 2
    in_end = min(L, g_last + Wb)
    o1 = min(L + N - 1, Np - 1 + b1 * W)
    if info["mode"] == MODE_XCORR:
        o1 = min(max(o1, N - 1), L) - (N - 1)
    return in_end, o1


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


class UnpackMarginWarning(RuntimeWarning):
    """PC_W_UNPACK_MARGIN: an FFT-core launch saw a last-digit residual above 0.25 LSB."""


def _check(rc, where):
    if rc == PC_W_UNPACK_MARGIN:
        import warnings
        warnings.warn(f"{where}: {status_string(rc)} ({rc})", UnpackMarginWarning, stacklevel=3)
        return rc
    if rc != PC_OK:
        raise PcError(rc, where)
    return rc


def status_string(code):
    return load().conv_status_string(int(code)).decode()


def opts_default(**kw):
    o = conv_opts()
    load().conv_opts_default(C.byref(o))
    for k, v in kw.items():
        if not hasattr(o, k):
            raise AttributeError(f"conv_opts has no field {k}")
        setattr(o, k, v)
    return o


def plan_create(L, N, W_block, mode=MODE_CONV, packing=PACK_SYM, Q=127, opts=None, **kw):
    o = opts if opts is not None else opts_default(**kw)
    h = C.c_void_p()
    _check(load().conv_plan_create(C.byref(h), int(L), int(N), int(W_block), int(mode), int(packing), int(Q),
                                   C.byref(o)), "conv_plan_create")
    return h


def plan_set_kernel(plan, k_dev, stream=None):
    w = "conv_plan_set_kernel"
    i = _geom(plan)
    return _check(load().conv_plan_set_kernel(plan, _dev(k_dev, i["N"], w, "k", i), _stream(stream)), w)


def execute(plan, s_dev, r_dev, stream=None):
    w = "conv_execute"
    i = _geom(plan)
    if not isinstance(s_dev, int) and not isinstance(r_dev, int) and s_dev is not None and r_dev is not None \
            and hasattr(s_dev, "data_ptr") and s_dev.data_ptr() == r_dev.data_ptr():
        _bad(w, "s and r must not overlap")
    return _check(load().conv_execute(plan, _dev(s_dev, i["L"], w, "s", i), _dev(r_dev, i["L_out"], w, "r", i),
                                      _stream(stream)), w)


def execute_blocks(plan, s_dev, s_offset, r_dev, r_offset, block_begin, block_end, stream=None):
    w = "conv_execute_blocks"
    i = _geom(plan)
    in_end, out_end = _block_span(i, int(block_begin), int(block_end))
    return _check(load().conv_execute_blocks(plan, _dev(s_dev, max(0, in_end - int(s_offset)), w, "s", i),
                                             int(s_offset), _dev(r_dev, max(0, out_end - int(r_offset)), w, "r", i),
                                             int(r_offset), int(block_begin), int(block_end), _stream(stream)), w)


def execute_batch(plan, s_dev, n_signals, s_stride, r_dev, r_stride, stream=None):
    w = "conv_execute_batch"
    i = _geom(plan)
    n = int(n_signals)
    return _check(load().conv_execute_batch(plan, _dev(s_dev, _rows(n, int(s_stride), i["L"]), w, "s", i), n,
                                            int(s_stride), _dev(r_dev, _rows(n, int(r_stride), i["L_out"]), w, "r", i),
                                            int(r_stride), _stream(stream)), w)


def execute_host(plan, s_host, r_host, stream=None):
    w = "conv_execute_host"
    i = _geom(plan)
    return _check(load().conv_execute_host(plan, _host(s_host, i["L"], w, "s"), _host(r_host, i["L_out"], w, "r"),
                                           _stream(stream)), w)


def execute_host_blocks(plan, s_host, s_offset, r_host, r_offset, block_begin, block_end, stream=None):
    """conv_execute_host on a rank's block range: s_host holds global samples [s_offset, ...),
    r_host receives global outputs [r_offset, ...) (host buffers)."""
    w = "conv_execute_host_blocks"
    i = _geom(plan)
    in_end, out_end = _block_span(i, int(block_begin), int(block_end))
    return _check(load().conv_execute_host_blocks(plan, _host(s_host, max(0, in_end - int(s_offset)), w, "s"),
                                                  int(s_offset), _host(r_host, max(0, out_end - int(r_offset)), w, "r"),
                                                  int(r_offset), int(block_begin), int(block_end), _stream(stream)), w)


def best_match(best_dev, n, score_dev=None, lag_dev=None, cand_dev=None, first_index=0, stream=None):
    """conv_best_match: {score, lag, index} of the largest score (ties: smallest index) into
    best_dev (3 doubles, device) over (score[i], lag[i], first_index + i) or the rows of cand."""
    w = "conv_best_match"
    n = int(n)
    for name, x, k, dt in (("best", best_dev, 3, "float64"), ("score", score_dev, n, "float64"),
                           ("lag", lag_dev, n, "int64"), ("cand", cand_dev, 3 * n, "float64")):
        if x is not None and not isinstance(x, int):
            if not x.is_cuda or str(x.dtype) != "torch." + dt or not x.is_contiguous() or x.numel() < k:
                _bad(w, f"{name} must be a contiguous CUDA {dt} tensor of >= {k} elements")
    return _check(load().conv_best_match(_ptr(score_dev), _ptr(lag_dev), _ptr(cand_dev), n, int(first_index),
                                         _ptr(best_dev), _stream(stream)), w)


def xcorr_max(plan, db_dev, n_signals, s_stride, score_dev, lag_dev, stream=None):
    w = "conv_xcorr_max"
    i = _geom(plan)
    n = int(n_signals)
    return _check(load().conv_xcorr_max(plan, _dev(db_dev, _rows(n, int(s_stride), i["L"]), w, "db", i), n,
                                        int(s_stride), _dev(score_dev, n, w, "score", i),
                                        _dev(lag_dev, n, w, "lag", i, dtype="int64"), _stream(stream)), w)


def set_kernels(plan, q_dev, n, q_stride, stream=None):
    """One kernel per pair (NEXT-3): n rows of N doubles, row stride q_stride (device)."""
    w = "conv_plan_set_kernels"
    i = _geom(plan)
    return _check(load().conv_plan_set_kernels(plan, _dev(q_dev, _rows(int(n), int(q_stride), i["N"]), w, "q", i),
                                               int(n), int(q_stride), _stream(stream)), w)


def xcorr_pairs(plan, x_dev, n, x_stride, score_dev, lag_dev, stream=None):
    """score/lag of pair i = (row i of x, kernel i); see include/packedconv.h."""
    w = "conv_xcorr_pairs"
    i = _geom(plan)
    n = int(n)
    return _check(load().conv_xcorr_pairs(plan, _dev(x_dev, _rows(n, int(x_stride), i["L"]), w, "x", i), n,
                                          int(x_stride), _dev(score_dev, n, w, "score", i),
                                          _dev(lag_dev, n, w, "lag", i, dtype="int64"), _stream(stream)), w)


def execute_debug(plan, s_dev, r_dev=None, packed=None, rbar=None, rint=None, c_s=None, stream=None,
                  max_residual=False):
    """Per-step dumps (see include/packedconv.h); returns the max last-digit residual (LSB) if
    max_residual, else None."""
    w = "conv_execute_debug"
    i = _geom(plan)
    P = i["P"]
    res = C.c_double(0.0)
    _check(load().conv_execute_debug(plan, _dev(s_dev, i["L"], w, "s", i),
                                     _dev(r_dev, i["L_out"], w, "r", i, optional=True),
                                     _dev(packed, P * i["packed_stride"], w, "packed", i, optional=True),
                                     _dev(rbar, P * i["rbar_stride"], w, "rbar", i, optional=True),
                                     _dev(rint, P * i["rint_stride"], w, "rint", i, dtype="int64", optional=True),
                                     _dev(c_s, P, w, "c_s", i, optional=True),
                                     C.byref(res) if max_residual else None, _stream(stream)), w)
    return res.value if max_residual else None


def adapt_block(plan, s_dev, snr_floor_db, calib_offset_db=0.0, P=None, stream=None):
    """Returns a list of (packing, Q, snr_lin) per block if P is given."""
    w = "conv_adapt_block"
    i = _geom(plan)
    out = (conv_block_decision * int(P))() if P else None
    _check(load().conv_adapt_block(plan, _dev(s_dev, i["L"], w, "s", i), float(snr_floor_db),
                                   float(calib_offset_db), out, _stream(stream)), w)
    return [(d.packing, d.Q, d.snr_lin) for d in out] if out is not None else None


def adapt_blocks(plan, s_dev, s_offset, block_begin, block_end, snr_floor_db, calib_offset_db=0.0,
                 want=False, stream=None):
    """conv_adapt_blocks on a shard: s_dev holds global samples [s_offset, ...).  Returns the
    decisions of blocks [block_begin, block_end) if want."""
    w = "conv_adapt_blocks"
    i = _geom(plan)
    b0, b1 = int(block_begin), int(block_end)
    in_end, _ = _block_span(i, b0, b1)
    out = (conv_block_decision * (b1 - b0))() if want and b1 > b0 else None
    _check(load().conv_adapt_blocks(plan, _dev(s_dev, max(0, in_end - int(s_offset)), w, "s", i), int(s_offset), b0,
                                    b1, float(snr_floor_db), float(calib_offset_db), out, _stream(stream)), w)
    return [(d.packing, d.Q, d.snr_lin) for d in out] if out is not None else None


def snr_calibrate(plan, s_dev, k_dev, Q=8, stream=None):
    """Single-point SNR-model calibration: returns (offset_db, measured_db, model_db)."""
    w = "conv_snr_calibrate"
    i = _geom(plan)
    off, meas, model = C.c_double(), C.c_double(), C.c_double()
    _check(load().conv_snr_calibrate(plan, _dev(s_dev, i["L"], w, "s", i), _dev(k_dev, i["N"], w, "k", i), int(Q),
                                     C.byref(off), C.byref(meas), C.byref(model), _stream(stream)), w)
    return off.value, meas.value, model.value


def execute_profile(plan, s_dev, r_dev, records_dev, stream=None):
    """Returns the persistent grid size; records_dev (uint64, 4*148*32) gets per-CTA
    {smid, t_start_ns, t_end_ns, blocks}."""
    w = "conv_execute_profile"
    i = _geom(plan)
    g = C.c_int32()
    _check(load().conv_execute_profile(plan, _dev(s_dev, i["L"], w, "s", i), _dev(r_dev, i["L_out"], w, "r", i),
                                       _ptr(records_dev), C.byref(g), _stream(stream)), w)
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
        _GEOM.pop(_handle(plan), None)
        load().conv_plan_destroy(plan)


_GEOM = {}   # plan handle -> its immutable geometry (L, L_out, P, N, strides, device): argument checks


def _handle(plan):
    return plan.value if isinstance(plan, C.c_void_p) else int(plan)


def _geom(plan):
    g = _GEOM.get(_handle(plan))
    if g is None:
        g = _GEOM[_handle(plan)] = plan_query(plan)
    return g


class Plan:
    """Owning wrapper: ``with Plan(L, N, W_block, ...) as p: p.set_kernel(k); p.execute(s, r)``."""

    def __init__(self, L, N, W_block, mode=MODE_CONV, packing=PACK_SYM, Q=127, **opts):
        self.h = None
        self.h = plan_create(L, N, W_block, mode, packing, Q, **opts)

    def set_kernel(self, k_dev, stream=None):
        plan_set_kernel(self.h, k_dev, stream)
        return self

    def execute(self, s_dev, r_dev, stream=None):
        return execute(self.h, s_dev, r_dev, stream)

    def execute_blocks(self, *a, **k):
        return execute_blocks(self.h, *a, **k)

    def execute_batch(self, *a, **k):
        return execute_batch(self.h, *a, **k)

    def execute_host(self, *a, **k):
        return execute_host(self.h, *a, **k)

    def execute_host_blocks(self, *a, **k):
        return execute_host_blocks(self.h, *a, **k)

    def execute_debug(self, *a, **k):
        return execute_debug(self.h, *a, **k)

    def xcorr_max(self, *a, **k):
        return xcorr_max(self.h, *a, **k)

    def set_kernels(self, *a, **k):
        return set_kernels(self.h, *a, **k)

    def xcorr_pairs(self, *a, **k):
        return xcorr_pairs(self.h, *a, **k)

    def adapt_block(self, s_dev, floor_db, calib_offset_db=0.0, stream=None):
        return adapt_block(self.h, s_dev, floor_db, calib_offset_db, self.info()["P"], stream)

    def adapt_blocks(self, *a, **k):
        return adapt_blocks(self.h, *a, **k)

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
