"""Critical-path breakdown of one option from an FL_TRACE build's chain event trace.
python tools/trace.py lib_trace.so [cfg] [n]   (traces work item 0 of the batch)"""
import ctypes, os, shutil, sys
from collections import defaultdict
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
shutil.copy(sys.argv[1], os.path.join(root, "paper_2303_02317_b200", "libfftlattice_b200.so"))
from paper_2303_02317_b200 import _native
from paper_2303_02317_b200.workloads import draw_config

cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 6
n = int(sys.argv[3]) if len(sys.argv) > 3 else 1
b = draw_config(cfg, n=n)
db = _native.DeviceBatch(b.kind, b.S, b.K, b.R, b.Y, b.V, b.E, b.T)
L = _native.lib()
L.fl_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int64]
CAP = 1 << 21
buf = np.zeros(CAP, dtype=np.uint64)
db.run(); db.fetch()
L.fl_trace_read(buf.ctypes.data, 1)  # reset
db.run(); db.fetch()
L.fl_trace_read(buf.ctypes.data, CAP)
cnt = int(buf[0])
ev = buf[1:1 + cnt].reshape(-1, 2)
typ = (ev[:, 0] >> np.uint64(32)).astype(np.int64)
arg = (ev[:, 0] & np.uint64(0xffffffff)).astype(np.int64)
clk = ev[:, 1].astype(np.int64)
names = {1: "SUB", 3: "LEAF", 5: "HWAIT", 7: "POST", 9: "CWAIT", 11: "ISSUE", 13: "STAGE", 16: "OPT", 18: "TWAIT"}
MARK = 20
print(f"events {len(typ)}  span {clk[-1] - clk[0]:.4g} cycles")
# innermost-open attribution
stack = []
acc = defaultdict(int)
gap = defaultdict(int)
prev_t, prev_e = clk[0], (typ[0], arg[0])
hw_by_q = defaultdict(int)
post_by = defaultdict(int)
leaf_n = 0
for t, a, c in zip(typ, arg, clk):
    dt = c - prev_t
    cat = stack[-1] if stack else "top"
    acc[cat] += dt
    def lab(e, a):
        if e == MARK: return f"M{a}"
        return names.get(e, names.get(e - 1, str(e))) + ("_B" if e in names else "_E")
    if cat in ("SUB", "top", "OPT"):
        gap[(cat, lab(*prev_e), lab(t, a))] += dt
    if cat == "HWAIT":
        hw_by_q[prev_e[1]] += dt
    if cat == "POST":
        post_by[prev_e[1] // 1024] += dt
    if t in names:
        stack.append(names[t])
    elif t - 1 in names:
        if stack and stack[-1] == names[t - 1]:
            stack.pop()
        if t == 4:
            leaf_n += 1
    prev_t, prev_e = c, (t, a)
tot = sum(acc.values())
print("innermost-category cycles:")
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"  {k:8s} {v:12.4g}  {100 * v / tot:5.1f}%")
print(f"leaves {leaf_n}")
print("helper waits by queue:", dict(hw_by_q))
print("posts by Lout:", {k: v for k, v in sorted(post_by.items())})
print("largest uncovered gaps (category, after, before): cycles")
for k, v in sorted(gap.items(), key=lambda kv: -kv[1])[:14]:
    print(f"  {k}: {v:.4g}")
