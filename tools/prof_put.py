"""Scheduler profile of one put batch (FL_PROFILE=1): per-role cycle counters."""
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
# must match the PROF_* enum in csrc/fl_sched.cuh
names = ["FFT_CYC", "FFT_N", "DIR_CYC", "DIR_N", "OTHER_CYC", "OTHER_N", "BIG_CYC", "BIG_N",
         "STRIP_CYC", "STRIP_ROWS", "WAIT_CYC", "FUSE_CYC", "FUSE_N", "KERNEL_CYC", "IDLE_CYC",
         "ISS_CYC", "CHAIN_CYC", "DEPWAIT_CYC", "ISS_SCAN", "ISS_STALL", "ISS_SLOT", "F_STAGE", "F_MID",
         "F_BOT", "STRIP_LOOP", "LEAF_LOAD", "W_RAW_S", "W_RAW_B", "W_WAR_S", "W_WAR_B", "W_N", "W_SUML", "W_SUMH", "W_FFT", "W_MAXL", "MAX_LOUT", "MAX_H", "MAX_YX", "HB64", "HB128", "HB256", "HB512", "HBBIG", "LB64", "LB128", "LB256", "LB512", "LBBIG"]
P = dict(zip(names, p[:len(names)]))
P["HELP_CYC"], P["HELP_CYC_BG"], P["HELP_FMA"], P["S_LEAF"] = p[48], p[49], p[50], p[51]
print(f"wall {1e3*(t1-t0):.2f} ms  n={n} cfg={cfg}")
for nm in names:
    print(f"{nm:12s} {P[nm]:.4g}")
nopt = n
d = lambda a, b: a / max(b, 1)
print("per option: chain %.3g cyc, strip %.3g cyc (%.0f rows), wait %.3g, fused %.3g (n=%.0f), issue %.3g"
      % (P["CHAIN_CYC"] / nopt, P["STRIP_CYC"] / nopt, P["STRIP_ROWS"] / nopt, P["WAIT_CYC"] / nopt,
         P["FUSE_CYC"] / nopt, P["FUSE_N"] / nopt, P["ISS_CYC"] / nopt))
print("small tasks: fft n=%.0f avg %.0f cyc; direct n=%.0f avg %.0f; other n=%.0f avg %.0f"
      % (P["FFT_N"], d(P["FFT_CYC"], P["FFT_N"]), P["DIR_N"], d(P["DIR_CYC"], P["DIR_N"]),
         P["OTHER_N"], d(P["OTHER_CYC"], P["OTHER_N"])))
print("big tasks: n=%.0f avg %.0f cyc" % (P["BIG_N"], d(P["BIG_CYC"], P["BIG_N"])))
ntask = P["FFT_N"] + P["DIR_N"] + P["OTHER_N"] + P["BIG_N"]
print("issue per task: scan %.0f stall %.0f slot %.0f (tasks/option %.0f)" % (
    d(P["ISS_SCAN"], ntask), d(P["ISS_STALL"], ntask), d(P["ISS_SLOT"], ntask), ntask / nopt))
print("fused per node: stage %.0f wait %.0f post %.0f leaf %.0f rest %.0f (of %.0f)" % (
    d(P["F_STAGE"], P["FUSE_N"]), d(P["F_MID"], P["FUSE_N"]), d(P["F_BOT"], P["FUSE_N"]), d(P["STRIP_CYC"], P["FUSE_N"]),
    d(P["FUSE_CYC"] - P["F_STAGE"] - P["F_MID"] - P["F_BOT"] - P["STRIP_CYC"], P["FUSE_N"]), d(P["FUSE_CYC"], P["FUSE_N"])))
print("strip: whole leaf %.1f cyc/row, row loop %.1f cyc/row, prologue %.1f cyc/row (per row of strip)" % (
    d(P["STRIP_CYC"], P["STRIP_ROWS"]), d(P["STRIP_LOOP"], P["STRIP_ROWS"]), d(P["LEAF_LOAD"], P["STRIP_ROWS"])))
print("conflict waits per option: RAW small %.3g big %.3g, WAR small %.3g big %.3g (n=%.0f)" % (
    P["W_RAW_S"] / nopt, P["W_RAW_B"] / nopt, P["W_WAR_S"] / nopt, P["W_WAR_B"] / nopt, P["W_N"] / nopt))
print("helpers: urgent %.3g cyc, background %.3g cyc per option; %.3g FMA per option (%.2f FMA/cycle)" % (
    P["HELP_CYC"] / nopt, P["HELP_CYC_BG"] / nopt, P["HELP_FMA"] / nopt,
    P["HELP_FMA"] / max(P["HELP_CYC"] + P["HELP_CYC_BG"], 1)))
print("status nonzero:", int(np.sum(r.status != 0)))
