"""Per-source-line stall summary of an ncu source-page CSV (--print-source cuda,sass).
python tools/ncu_lines.py src.csv [file-substring] [top]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
cur, hdr, out = None, None, []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1]; continue
    if r and r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}; continue
    if not r or not r[0] or hdr is None or not r[0].isdigit():
        continue
    def g(k):
        try: return float(r[hdr[k]])
        except Exception: return 0.0
    out.append((cur.split("/")[-1], int(r[0]), r[1].strip()[:70], g("Warp Stall Sampling (All Samples)"),
                g("stall_no_inst"), g("stall_long_sb"), g("stall_short_sb"), g("stall_wait"), g("stall_sleep"),
                g("stall_branch_resolving"), g("Instructions Executed")))
tot = sum(o[3] for o in out)
print(f"total samples {tot:.0f}")
by = {}
for o in out:
    by[o[0]] = by.get(o[0], 0) + o[3]
print({k: round(v) for k, v in sorted(by.items(), key=lambda kv: -kv[1])})
sel = [o for o in out if want in o[0]]
sel.sort(key=lambda o: -o[3])
print("file:line samples no_inst long_sb short_sb wait sleep branch exec | source")
for o in sel[:top]:
    print(f"{o[0]}:{o[1]} {o[3]:.0f} {o[4]:.0f} {o[5]:.0f} {o[6]:.0f} {o[7]:.0f} {o[8]:.0f} {o[9]:.0f} {o[10]:.3g} | {o[2]}")
