"""Scheduler profile of one put batch (FL_PROFILE=1)."""
import os, sys, time
os.environ["FL_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2303_02317_b200 import _native
from paper_2303_02317_b200.workloads import draw_config
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 6
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
b = draw_config(cfg, n=n)
db = _native.DeviceBatch(b.kind, b.S, b.K, b.R, b.Y, b.V, b.E, b.T)
db.run(); db.fetch()
t0 = time.perf_counter(); db.run(); r = db.fetch(); t1 = time.perf_counter()
p = db.profile().astype(np.float64)
names = ["FFT_CYC","FFT_N","DIR_CYC","DIR_N","KB_CYC","KB_N","OTHER_CYC","OTHER_N","STRIP_CYC","STRIP_ROWS","WAIT_CYC","WAIT_N","ROWLOOP_CYC","KERNEL_CYC","IDLE_CYC","FFT_LOUT","DIR_LOUT","CHAIN_CYC","LOADS_CYC","DIVERGED"]
print(f"wall {1e3*(t1-t0):.2f} ms  n={n} cfg={cfg}")
for i, nm in enumerate(names):
    print(f"{nm:12s} {p[i]:.4g}")
nopt = n
print("per option: strip rows %.0f, strip cyc %.3g, wait cyc %.3g, chain cyc %.3g" % (p[9]/nopt, p[8]/nopt, p[10]/nopt, p[17]/nopt))
print("per task: fft %.0f cyc (n=%d, Lout avg %.0f), direct %.0f cyc (n=%d), kbuild %.0f (n=%d)" % (p[0]/max(p[1],1), p[1], p[15]/max(p[1],1), p[2]/max(p[3],1), p[3], p[4]/max(p[5],1), p[5]))
print("worker busy frac: %.3f" % ((p[0]+p[2]+p[4]+p[6]) / max(p[13],1)))
