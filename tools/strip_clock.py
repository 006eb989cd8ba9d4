"""Chain time split in the kernel from a FL_STRIP_CLOCK=1 build (a few clock64
intervals, nothing else instrumented): python tools/strip_clock.py n [cfg]"""
import os, sys
os.environ["FL_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_02317_b200 import _native
from paper_2303_02317_b200.workloads import draw_config
n = int(sys.argv[1]); cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 6
b = draw_config(cfg, n=n)
db = _native.DeviceBatch(b.kind, b.S, b.K, b.R, b.Y, b.V, b.E, b.T)
db.run(); db.fetch()
db.run(); r = db.fetch()
p = [float(v) for v in db.profile()]
# slots: fl_sched.cuh PROF_* enum
STRIP_CYC, STRIP_N, WAIT, FUSE, FUSE_N, CHAIN, STAGE, HWAIT, HPOST, LOOP = 8, 9, 10, 11, 12, 16, 21, 22, 23, 24
rows = max(p[STRIP_N], 1)
ch = p[CHAIN] / n
print(f"n={n}: chain {ch:.3g} cycles/option; per option: strip loop {p[LOOP]/n:.3g} ({p[LOOP]/rows:.0f}/row), "
      f"leaf other {(p[STRIP_CYC]-p[LOOP])/n:.3g}, subtree entry wait {p[WAIT]/n:.3g}, staging {p[STAGE]/n:.3g}, "
      f"helper waits {p[HWAIT]/n:.3g}, helper posts {p[HPOST]/n:.3g}, "
      f"walk rest {(p[FUSE]-p[STAGE]-p[HWAIT]-p[HPOST]-p[STRIP_CYC])/n:.3g}, "
      f"above subtrees {(p[CHAIN]-p[FUSE]-p[WAIT])/n:.3g}  ({p[FUSE_N]/n:.0f} subtrees)")
print(f"  options re-priced on the full frame: {int(p[51])} of {n}")
print(f"  above subtrees: option setup {p[17] / n:.3g}, jump issue (chain_conv) {p[15] / n:.3g}, "
      f"residual wait (calls) {p[25] / n:.3g} cycles/option")
for r, nm in enumerate(["small", "big", "low"]):
    q, sv, cnt, st = p[36 + 4 * r: 40 + 4 * r]
    if cnt:
        print(f"  ring {nm}: {cnt / n:.0f} tasks/option, queue {q / cnt:.0f} cycles, service {sv / cnt:.0f} cycles"
              + (f", {100 * st / cnt:.0f} % run by the big group" if r == 0 else ""))
print("  issued per option by ring (small, big, low):", [round(p[48 + r] / n) for r in range(3)],
      " with no dependency at issue:", [round(p[52 + r] / n) for r in range(3)])
