"""Per-option timeline of one batch (FL_PROFILE=1): makespan, option durations,
and how busy the SMs / chain slots are.  python tools/timeline.py [cfg] [n] [lib.so]"""
import os, sys
os.environ["FL_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
if len(sys.argv) > 3:
    import shutil
    shutil.copy(sys.argv[3], os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                          "paper_2303_02317_b200", "libfftlattice_b200.so"))
from paper_2303_02317_b200 import _native
from paper_2303_02317_b200.workloads import draw_config

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 6
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
b = draw_config(cfg, n=n)
db = _native.DeviceBatch(b.kind, b.S, b.K, b.R, b.Y, b.V, b.E, b.T)
db.run(); db.fetch()
db.run(); db.fetch()
tl = db.timeline().astype(np.int64)
t0 = tl[:, 0].min()
st, en = (tl[:, 0] - t0) / 1e6, (tl[:, 1] - t0) / 1e6
dur = en - st
sm, ch = tl[:, 2] >> 1, tl[:, 2] & 1
print(f"makespan {en.max():.3f} ms  (last start {st.max():.3f} ms)")
q = np.percentile(dur, [0, 10, 50, 90, 100])
print("option ms: min %.2f p10 %.2f med %.2f p90 %.2f max %.2f" % tuple(q))
per_sm = {}
for s_, d_ in zip(sm, dur):
    per_sm.setdefault(int(s_), []).append(d_)
two = [max(v) for v in per_sm.values() if len(v) >= 2]
one = [max(v) for v in per_sm.values() if len(v) == 1]
print(f"SMs used {len(per_sm)}: with >=2 options {len(two)} (max-option mean {np.mean(two) if two else 0:.2f} ms), "
      f"with 1 option {len(one)} (mean {np.mean(one) if one else 0:.2f} ms)")
order = np.argsort(-en)[:5]
for i in order:
    others = [j for j in range(len(sm)) if sm[j] == sm[i] and j != i]
    print(f"  late item {i}: T={int(b.T[i]) if i < len(b.T) else -1} sm {sm[i]} chain {ch[i]} start {st[i]:.2f} "
          f"dur {dur[i]:.2f}  co-resident {[(j, round(dur[j], 2)) for j in others]}")
