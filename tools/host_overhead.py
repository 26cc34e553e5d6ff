"""Is the bench host-bound?  Time K launches: (a) with per-step events, (b) without,
(c) host-side enqueue time per call."""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_1201_3018_b200 import binding as pcb
from paper_1201_3018_b200 import workloads as WL
s, k = WL.cfg2(seed=0)
dev = torch.device("cuda")
S = [torch.from_numpy(s).to(dev) for _ in range(4)]
R = [torch.empty(len(s) + len(k) - 1, dtype=torch.float64, device=dev) for _ in range(4)]
with pcb.Plan(len(s), len(k), 4096, 0, 2, 511, rmax_rule=1) as p:
    p.set_kernel(torch.from_numpy(k).to(dev))
    for i in range(5): p.execute(S[i % 4], R[i % 4])
    torch.cuda.synchronize()
    K = 100
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); t0 = time.perf_counter()
    for i in range(K): p.execute(S[i % 4], R[i % 4])
    t1 = time.perf_counter(); b.record(); torch.cuda.synchronize()
    print("no events: gpu %.1f us/step, host enqueue %.1f us/step" % (a.elapsed_time(b) / K * 1e3, (t1 - t0) / K * 1e6))
    st = torch.cuda.current_stream().cuda_stream
    h = p.h
    lib = pcb.load()
    ptrs = [(S[i % 4].data_ptr(), R[i % 4].data_ptr()) for i in range(K)]
    a.record(); t0 = time.perf_counter()
    for i in range(K): lib.conv_execute(h, ptrs[i][0], ptrs[i][1], st)
    t1 = time.perf_counter(); b.record(); torch.cuda.synchronize()
    print("raw ctypes: gpu %.1f us/step, host enqueue %.1f us/step" % (a.elapsed_time(b) / K * 1e3, (t1 - t0) / K * 1e6))
    # host-ahead: enqueue a long sleep kernel first so the queue is full
    torch.cuda._sleep(50_000_000)
    a.record()
    for i in range(K): lib.conv_execute(h, ptrs[i][0], ptrs[i][1], st)
    b.record(); torch.cuda.synchronize()
    print("queue pre-filled: gpu %.1f us/step" % (a.elapsed_time(b) / K * 1e3))
