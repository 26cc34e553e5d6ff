import json, numpy as np, sys
import torch
sys.path.insert(0, '.')
from paper_1201_3018_b200 import binding as pcb
from paper_1201_3018_b200 import workloads as WL
dev = torch.device('cuda')
s, k = WL.cfg2(seed=0, L=1 << 22)
S = torch.from_numpy(s).to(dev); R = torch.empty(len(s) + len(k) - 1, dtype=torch.float64, device=dev)
NC = 148 * 32; KTW = 24 * NC; KTP = KTW + 148 * 16 * 16 * 4
rec = torch.zeros(KTP + 148 * 4 * 16 * 4, dtype=torch.int64, device=dev)
o = pcb.opts_default(rmax_rule=1)
with pcb.Plan(len(s), len(k), 4096, 0, 2, 511, opts=o) as p:
    p.set_kernel(torch.from_numpy(k).to(dev))
    for _ in range(3): p.execute(S, R)
    rec.zero_(); g = pcb.execute_profile(p.h, S, R, rec); torch.cuda.synchronize()
a = rec.cpu().numpy()
r = a[:4 * g].reshape(g, 4)
t0 = r[:, 1].min(); en = (r[:, 2] - t0) / 1e3
Pr = a[KTP:KTP + 148 * 4 * 16 * 4].reshape(148, 4, 16, 4)[:g]
jobs = []
for c in range(g):
    n = 0
    for w in range(4):
        for j in range(15):
            if Pr[c, w, j, 3]:
                n += 1
    jobs.append(n)
jobs = np.array(jobs)
# producer records include sentinels: count real = published minus sentinel sequences (~3)
print('published per CTA hist', np.bincount(jobs).tolist())
for n in sorted(set(jobs)):
    m = jobs == n
    print(n, 'ctas', m.sum(), 'end us min/med/max', round(en[m].min(),1), round(np.median(en[m]),1), round(en[m].max(),1))
