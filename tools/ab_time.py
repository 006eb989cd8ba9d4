"""A/B timing of library builds on the headline batch: python tools/ab_time.py lib1.so lib2.so ...
(binds only the batch entry points, so older builds load too)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2303_02317_b200.workloads import draw_config

b = draw_config(int(os.environ.get('AB_CFG', 6)), n=int(os.environ.get('AB_N', 256)))
P, i64, i32, d, c_int = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_int
ptr = lambda a: a.ctypes.data_as(P)
kind = np.ascontiguousarray(b.kind, dtype=np.int8)
T = np.ascontiguousarray(b.T, dtype=np.int64)
arrs = [np.ascontiguousarray(getattr(b, f), dtype=np.float64) for f in "SKRYVE"]
torch.cuda.init()
for path in sys.argv[1:]:
    L = ctypes.CDLL(os.path.abspath(path))
    L.fl_batch_prepare.argtypes = [ctypes.POINTER(P), i64, P, P, P, P, P, P, P, P, d, i64, i64, c_int, i32, P]
    L.fl_batch_run.argtypes = [P, P]
    L.fl_batch_fetch.argtypes = [P, P, P, P, P, P, P]
    L.fl_batch_free.argtypes = [P]
    h = P()
    assert L.fl_batch_prepare(ctypes.byref(h), len(kind), ptr(kind), *[ptr(a) for a in arrs], ptr(T), 0.4, 256, 128, 0, 0, None) == 0
    price = np.empty(len(kind)); st = np.empty(len(kind), dtype=np.int32)
    for _ in range(3):
        L.fl_batch_run(h, None)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); L.fl_batch_run(h, None); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    L.fl_batch_fetch(h, ptr(price), ptr(st), None, None, None, None)
    print(f"{os.path.basename(path)}: {np.mean(ts):.3f} ms (min {min(ts):.3f})  errors {int(np.sum(st != 0))}  p0 {price[0]:.15g}")
    L.fl_batch_free(h)
