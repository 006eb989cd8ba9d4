"""Per-option chain durations of one batch (FL_PROF build, FL_PROFILE=1):
distribution, and how the makespan compares with the mean."""
import os, sys
os.environ["FL_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2303_02317_b200 import _native
from paper_2303_02317_b200.workloads import draw_config
from paper_2303_02317_b200.shard import option_cost
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 6
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
b = draw_config(cfg, n=n)
db = _native.DeviceBatch(b.kind, b.S, b.K, b.R, b.Y, b.V, b.E, b.T)
db.run(); db.fetch(); db.run(); db.fetch()
tl = db.timeline().astype(np.float64)
st, en = tl[:, 0], tl[:, 1]
t0 = st.min()
dur = (en - st) / 1e6
print(f"makespan {(en.max() - t0) / 1e6:.3f} ms; per-option chain ms: min {dur.min():.3f} p10 {np.percentile(dur, 10):.3f} "
      f"median {np.median(dur):.3f} p90 {np.percentile(dur, 90):.3f} max {dur.max():.3f}")
print(f"start spread {(st.max() - t0) / 1e6:.3f} ms; end: p10 {(np.percentile(en, 10) - t0) / 1e6:.3f} median {(np.median(en) - t0) / 1e6:.3f} max {(en.max() - t0) / 1e6:.3f}")
# does the per-item work-item index (cost order) correlate with duration?
c = option_cost(b.kind, b.T)
sm = (tl[:, 2].astype(np.int64) >> 1)
print("corr(duration, ks) =", np.corrcoef(dur, b.S / b.K)[0, 1])
pairs = {}
for i in range(n):
    pairs.setdefault(int(sm[i]), []).append(i)
solo = [v for v in pairs.values() if len(v) == 1]
two = [v for v in pairs.values() if len(v) == 2]
print(f"SMs used {len(pairs)}: solo {len(solo)}, paired {len(two)}")
if solo:
    print(f"solo durations mean {np.mean([dur[v[0]] for v in solo]):.3f}; paired mean {np.mean([dur[i] for v in two for i in v]):.3f}")
if os.environ.get("TL_SAVE"):
    np.savez(os.environ["TL_SAVE"], dur=dur, S=b.S, K=b.K, R=b.R, Y=b.Y, V=b.V, E=b.E, T=b.T, sm=sm, start=st, end=en)
