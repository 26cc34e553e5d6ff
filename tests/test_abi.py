"""CPU-side checks of the C-ABI boundary: the library builds/loads, exports every symbol
include/packedconv.h declares, the ctypes structs match the C layout, and without a GPU
every compute entry point fails loudly (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "packedconv.h")


@pytest.fixture(scope="module")
def lib():
    from paper_1201_3018_b200 import build as B
    B.build_library()
    from paper_1201_3018_b200 import binding
    return binding.load()


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(conv_\w+)\s*\(", txt, flags=re.M)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("conv_plan_create", "conv_plan_set_kernel", "conv_execute", "conv_adapt_block",
                     "conv_execute_debug", "conv_plan_query", "conv_plan_destroy", "conv_status_string"):
        assert required in names


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib._name], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(\w+)", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing
    for n in declared_functions():
        getattr(lib, n)


def test_struct_layout_matches_c(lib):
    """Every named field of the ctypes mirrors sits at the C offset (no magic reserved[] slots)."""
    from paper_1201_3018_b200 import binding as b
    structs = [("conv_opts", b.conv_opts), ("conv_plan_info", b.conv_plan_info), ("conv_shard", b.conv_shard),
               ("conv_block_decision", b.conv_block_decision)]
    lines, want = [], []
    for cname, cls in structs:
        lines.append(f'printf("%zu\\n", sizeof({cname}));')
        want.append(C.sizeof(cls))
        for fname, _ in cls._fields_:
            lines.append(f'printf("%zu\\n", offsetof({cname}, {fname}));')
            want.append(getattr(cls, fname).offset)
    src = "#include <stdio.h>\n#include <stddef.h>\n#include \"packedconv.h\"\nint main(void) {\n" + \
        "\n".join(lines) + "\nreturn 0;\n}\n"
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "t")
        subprocess.check_call(["gcc", "-I", os.path.dirname(HEADER), c, "-o", exe])
        vals = [int(v) for v in subprocess.check_output([exe]).split()]
    assert vals == want
    # the tuning knobs are named fields, not reserved slots
    names = [f for f, _ in b.conv_opts._fields_]
    for f in ("fft_n", "core_variant", "core_tile", "parts_per_job", "unpack_form", "validate_trials"):
        assert f in names
    assert "reserved" not in names


def test_library_reads_no_environment(lib):
    """Library behaviour is set through conv_opts only: no getenv in the sources."""
    csrc = os.path.join(ROOT, "paper_1201_3018_b200", "csrc")
    for f in os.listdir(csrc):
        assert "getenv" not in open(os.path.join(csrc, f)).read(), f


def test_release_kernels_do_not_trap(lib):
    """The persistent kernel's watchdog raises a host-mapped flag and exits (PC_E_WATCHDOG) in
    release builds; __trap (a sticky context error) exists only in PC_DEBUG_TRAP builds."""
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib._name], capture_output=True,
                          text=True).stdout
    assert "BPT.TRAP" not in sass


def test_binding_rejects_bad_buffers():
    """The C ABI takes no lengths: the binding checks dtype, contiguity, device and size."""
    import torch
    from paper_1201_3018_b200 import binding as b
    info = {"device": 0, "L": 100, "N": 9, "Np": 9, "W": 30, "W_block": 40, "mode": b.MODE_CONV}
    with pytest.raises(b.PcError) as ei:
        b._dev(torch.zeros(100, dtype=torch.float64), 100, "w", "s", info)      # host tensor
    assert ei.value.code == b.PC_E_CONFIG
    with pytest.raises(b.PcError):
        b._host(np_zeros(50), 100, "w", "s")                                     # too short
    with pytest.raises(b.PcError):
        b._host(np_zeros(200).astype("float32"), 100, "w", "s")                  # wrong dtype
    with pytest.raises(b.PcError):
        b._host(np_zeros(400)[::2], 100, "w", "s")                               # strided
    assert b._host(np_zeros(100), 100, "w", "s")
    assert b._dev(12345, 10**9, "w", "s", info) == 12345                         # raw pointer: caller-managed
    # block spans (reading C7, Eq. (17)): blocks [0, 2) of L = 100, N' = 9, W = 30, W_block = 40
    assert b._block_span(info, 0, 2) == (min(100, 30 - 2 + 40), 9 - 1 + 60)
    assert b._block_span(info, 1, 4) == (100, 100 + 9 - 1)


def np_zeros(n):
    import numpy as np
    return np.zeros(n)


def test_status_strings_and_defaults(lib):
    from paper_1201_3018_b200 import binding as b
    assert b.status_string(0) == "ok"
    assert "bound" in b.status_string(b.PC_E_BOUND)
    o = b.opts_default()
    assert o.eps_rule == b.EPS_POW2 and o.rmax_rule == b.RMAX_PAPER and o.u_sys == 3.1193e-11


def test_no_cpu_fallback_without_gpu(lib):
    """On a box without a CUDA device, plan creation reports PC_E_CUDA (no silent CPU path)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1201_3018_b200 import binding as b
    with pytest.raises(b.PcError) as ei:
        b.plan_create(1000, 9, 40, b.MODE_CONV, b.PACK_SYM, 7)
    assert ei.value.code == b.PC_E_CUDA


def test_config_errors_precede_device_checks(lib):
    from paper_1201_3018_b200 import binding as b
    for args in ((0, 9, 40), (1000, 0, 40), (1000, 9, 12), (1000, 9, 27)):
        with pytest.raises(b.PcError) as ei:
            b.plan_create(*args, b.MODE_CONV, b.PACK_SYM, 7)
        assert ei.value.code == b.PC_E_CONFIG


def test_library_has_sm100a_code_and_tma(lib):
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib._name], capture_output=True,
                          text=True).stdout
    assert "sm_100a" in subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", lib._name], capture_output=True,
                                       text=True).stdout
    assert "DFMA" in sass
    assert "UBLKCP" in sass           # cp.async.bulk (TMA bulk copy) staging of blocks/taps


def _build_c_example(lib, out):
    src = os.path.join(ROOT, "examples", "conv_example.c")
    libdir = os.path.dirname(lib._name)
    subprocess.check_call(["gcc", "-O2", "-I", os.path.join(ROOT, "include"), src, "-o", out,
                           "-L", "/usr/local/cuda/lib64", "-lcudart", "-L", libdir, "-lpackedconv",
                           f"-Wl,-rpath,{libdir}", "-Wl,-rpath,/usr/local/cuda/lib64", "-lm"])


def test_c_example_builds_against_the_abi(lib):
    """A plain C program (examples/conv_example.c) compiles and links against include/packedconv.h
    and the library alone -- the boundary needs no Python."""
    with tempfile.TemporaryDirectory() as d:
        _build_c_example(lib, os.path.join(d, "conv_example"))


@pytest.mark.gpu
def test_c_example_runs(lib):
    """The C example runs the packed path end to end through host buffers and meets 40 dB."""
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "conv_example")
        _build_c_example(lib, exe)
        out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
        assert out.returncode == 0, out.stdout + out.stderr
        assert "SNR vs full precision" in out.stdout
