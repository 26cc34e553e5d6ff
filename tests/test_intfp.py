"""The producer warps' integer-pipe binary64 arithmetic (paper_1201_3018_b200/csrc/pc_intfp.cuh)
is bit-identical to the host's IEEE FP64 arithmetic: RN products and quotients of positive
normals, Eq. (2)'s round-half-away companding (reading C5) and the Eqs. (4)/(7) packed
words under the dyadic eps (reading C4), including exact ties and negative zeros.
The header is host-compilable; this builds tests/intfp_check.cpp with g++ and runs it."""
import os
import shutil
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_intfp_bit_identical_to_fp64(tmp_path):
    exe = str(tmp_path / "intfp_check")
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-o", exe,
                    os.path.join(HERE, "intfp_check.cpp")], check=True)
    res = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    assert " fails 0" in res.stdout
