"""e2e (host buffers) timing of the cfg2 asym2 point: conv_execute_host vs the shard form, with
and without an initialised NCCL process group (diagnostics)."""
import os
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1201_3018_b200 import binding as pcb
from paper_1201_3018_b200 import workloads as WL

s, k = WL.cfg2(seed=0)
dev = torch.device("cuda")
if len(sys.argv) > 1 and sys.argv[1] == "pg":
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533", RANK="0", WORLD_SIZE="1")
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
with pcb.Plan(len(s), len(k), 4096, 0, 2, 511, rmax_rule=1) as p:
    p.set_kernel(torch.from_numpy(k).to(dev))
    sh = torch.from_numpy(s).pin_memory()
    rh = torch.empty(p.info()["L_out"], dtype=torch.float64).pin_memory()
    for name, f in (("host", lambda: p.execute_host(sh, rh)),
                    ("host_blocks", lambda: p.execute_host_blocks(sh, 0, rh, 0, 0, p.info()["P"]))):
        for _ in range(3):
            f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record()
        for _ in range(20):
            f()
        e1.record()
        torch.cuda.synchronize()
        print(name, sys.argv[1:], "event ms/step", e0.elapsed_time(e1) / 20, "wall", (time.perf_counter() - t0) / 20 * 1e3)
