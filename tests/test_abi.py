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
    from paper_1201_3018_b200 import binding as b
    src = r'''
#include <stdio.h>
#include <stddef.h>
#include "packedconv.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu\n", sizeof(conv_opts), offsetof(conv_opts, u_sys), sizeof(conv_plan_info),
         offsetof(conv_plan_info, eps), offsetof(conv_plan_info, q_mode), sizeof(conv_block_decision));
  return 0;
}
'''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "t")
        subprocess.check_call(["gcc", "-I", os.path.dirname(HEADER), c, "-o", exe])
        vals = [int(v) for v in subprocess.check_output([exe]).split()]
    want = [C.sizeof(b.conv_opts), b.conv_opts.u_sys.offset, C.sizeof(b.conv_plan_info), b.conv_plan_info.eps.offset,
            b.conv_plan_info.q_mode.offset, C.sizeof(b.conv_block_decision)]
    assert vals == want


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
