import json, sys, torch
sys.path.insert(0, ".")
n = 4 << 20
sh = torch.randn(n, dtype=torch.float64).pin_memory()
rh = torch.empty(n, dtype=torch.float64).pin_memory()
d_in = torch.empty(n, dtype=torch.float64, device="cuda")
d_out = torch.randn(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
res = {}
for wts in ([1]*8, [1,1]+[2]*11+[1,1], [1]*2):
    cum=[0]
    for w in wts: cum.append(cum[-1]+w)
    for rep in range(4):
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True); t0.record()
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur); s2.wait_stream(cur)
        ev=[]
        for c in range(len(wts)):
            a, b = n*cum[c]//cum[-1], n*cum[c+1]//cum[-1]
            t = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            with torch.cuda.stream(s1):
                t[0].record(); d_in[a:b].copy_(sh[a:b], non_blocking=True); t[1].record()
            s2.wait_event(t[1])
            with torch.cuda.stream(s2):
                t[2].record(); rh[a:b].copy_(d_out[a:b], non_blocking=True); t[3].record()
            ev.append((t, (b-a)*8))
        cur.wait_stream(s1); cur.wait_stream(s2)
        t1 = torch.cuda.Event(enable_timing=True); t1.record()
        torch.cuda.synchronize()
    res[str(len(wts))] = {"total_ms": round(t0.elapsed_time(t1),4),
        "chunks[h2d_s,h2d_e,d2h_s,d2h_e,MB]": [[round(t0.elapsed_time(e)*1e3,1) for e in t]+[round(nb/1e6,2)] for t,nb in ev]}
print(json.dumps(res, indent=0))
