"""Top CUDA source lines of an ncu report by warp-stall samples, with the dominant stall reasons
(ncu -i REP --page source --csv --print-source cuda,sass > CSV; python tools/ncu_source_lines.py CSV [N] [file-substring])."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
filt = sys.argv[3] if len(sys.argv) > 3 else ""
cur, hdr, out = None, None, []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0] or not r[0].isdigit():
        continue
    d = dict(zip(hdr[4:], r[4:]))
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    stalls = {k[6:]: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v.isdigit() and int(v)}
    out.append((s, cur.split("/")[-1], int(r[0]), r[1].strip()[:70], sorted(stalls.items(), key=lambda x: -x[1])[:4],
                d.get("Instructions Executed", "")))
tot = sum(o[0] for o in out)
print("total samples", tot)
for s, f, ln, src, st, ie in sorted([o for o in out if filt in o[1]], key=lambda x: -x[0])[:top]:
    print(f"{100 * s / tot:5.1f}% {f}:{ln} inst={ie} {src} | {st}")
