import sys, os, shutil, numpy as np
sys.path.insert(0, '.')
lib = sys.argv[1]
shutil.copy(lib, 'paper_2303_02317_b200/libfftlattice_b200.so')
from paper_2303_02317_b200 import _native
rows = [(S, 100.0, R, V, E, T) for (R, V) in ((1e-6, 0.6), (1e-5, 0.6), (1e-6, 0.1), (0.05, 0.3))
        for (S, E) in ((100.0, 365.0), (80.0, 500.0)) for T in (1024, 4096, 5000)]
S, K, R, V, E, T = (np.array([r[i] for r in rows]) for i in range(6))
T = T.astype(np.int64)
kind = np.full(len(rows), 2, dtype=np.int8)
res = _native.price_batch_full(kind, S, K, R, np.zeros(len(rows)), V, E, T, method=0, bnd_cap=64)
print(lib, [hex(int(s)) for s in res.status], res.price[:6])
