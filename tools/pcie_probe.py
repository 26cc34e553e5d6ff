"""PCIe copy bandwidth: H2D alone, D2H alone, both concurrently (pinned buffers)."""
import torch
n = 4 << 20
h_in = torch.randn(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.randn(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)
def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = timeit(fn)
    nb = 8 * n * (2 if name == "both" else 1)
    print(f"{name}: {ms:.3f} ms  {nb / ms / 1e6:.1f} GB/s")

# the conv_execute_host pipeline shape without the kernels: n chunks, H2D on s1, D2H on s2
# (chunk c's D2H after chunk c's H2D), 32 MB each way
for nchk in (1, 2, 4, 8, 16):
    ev = [torch.cuda.Event() for _ in range(nchk)]
    def pipe():
        csz = n // nchk
        for c in range(nchk):
            with torch.cuda.stream(s1):
                d_a[c * csz:(c + 1) * csz].copy_(h_in[c * csz:(c + 1) * csz], non_blocking=True)
                ev[c].record(s1)
            with torch.cuda.stream(s2):
                s2.wait_event(ev[c])
                h_out[c * csz:(c + 1) * csz].copy_(d_b[c * csz:(c + 1) * csz], non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
    ms = timeit(pipe)
    print(f"pipeline chunks={nchk}: {ms:.3f} ms")
