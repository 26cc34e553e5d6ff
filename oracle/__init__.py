"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct NumPy (float64 / int64) implementation of the hot path of
Anam & Andreopoulos, "Throughput Scaling Of Convolution For Error-Tolerant Multimedia
Applications" (arXiv 1201.3018; /root/reference/PAPER.md, cited as P:<line>).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything from here.  The product path
(``paper_1201_3018_b200``) never imports it and shares no code, header, table or
constant generator with it.  See oracle/packedconv.py for the per-function citations
and DESIGN.md §3 for the readings of the paper it follows.
"""
from .packedconv import *  # noqa: F401,F403
