"""Per-CUDA-source-line metrics from an ncu source export with
--print-source cuda,sass:  python tools/ncu_src_lines.py src.csv [sortkey] [top]
sortkey: samples | wave | excess | inst"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
key = sys.argv[2] if len(sys.argv) > 2 else "samples"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
cur, hdr, out = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        hdr = {}
        for i, k in enumerate(r):
            hdr.setdefault(k, i)
        continue
    if hdr is None or not r[0].isdigit():
        continue
    def g(k):
        try: return float(r[hdr[k]])
        except Exception: return 0.0
    out.append(dict(file=cur, line=int(r[0]), src=r[1].strip()[:80], samples=g("Warp Stall Sampling (All Samples)"),
                    wave=g("L1 Wavefronts Shared"), excess=g("L1 Wavefronts Shared Excessive"),
                    inst=g("Instructions Executed")))
tot = {k: sum(o[k] for o in out) for k in ("samples", "wave", "excess", "inst")}
print("totals", {k: f"{v:.4g}" for k, v in tot.items()})
byf = {}
for o in out:
    d = byf.setdefault(o["file"], {"samples": 0, "wave": 0, "excess": 0, "inst": 0})
    for k in d: d[k] += o[k]
for f, d in sorted(byf.items(), key=lambda kv: -kv[1][key]):
    print(f"{f:20s} " + " ".join(f"{k}={v:.3g}" for k, v in d.items()))
out.sort(key=lambda o: -o[key])
for o in out[:top]:
    print(f"{o['file']}:{o['line']} samples={o['samples']:.0f} wave={o['wave']:.3g} excess={o['excess']:.3g} inst={o['inst']:.3g} | {o['src']}")
