"""Hot local-memory (LDL/STL) instructions of an ncu source export
(--print-source cuda,sass): python tools/ncu_local.py src.csv [top]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur = hdr = srcline = None
out = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split('/')[-1]; continue
    if r[0] == "Line No":
        hdr = {}
        for i, k in enumerate(r):
            hdr.setdefault(k, i)
        continue
    if hdr is None:
        continue
    if r[0].isdigit():
        srcline = (cur, r[0], r[1].strip()[:70]); continue
    if r[0] == '' and len(r) > 3 and ('LDL' in r[3] or 'STL' in r[3]):
        ex = float(r[hdr["Instructions Executed"]] or 0)
        s = float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        out.append((ex, s, srcline, r[3].strip()))
out.sort(key=lambda o: -o[1])
print("LDL/STL sites", len(out), "executed", f"{sum(o[0] for o in out):.3g}", "samples", sum(o[1] for o in out))
for o in out[:top]:
    print(f"{o[0]:10.3g} {o[1]:6.0f} {o[2][0]}:{o[2][1]} {o[3][:36]:36s} | {o[2][2]}")
