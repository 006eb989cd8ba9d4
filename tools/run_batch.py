import os, sys
sys.path.insert(0, os.getcwd())
from paper_2303_02317_b200 import _native
from paper_2303_02317_b200.workloads import draw_config
b = draw_config(6, n=256)
db = _native.DeviceBatch(b.kind, b.S, b.K, b.R, b.Y, b.V, b.E, b.T)
for _ in range(2):
    db.run(); db.fetch()
print("ok")
