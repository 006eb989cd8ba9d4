#!/bin/bash
# Compare warp layouts (tools/bin/lib_layout*.so) on the headline put batch.
for L in "$@"; do
  cp tools/bin/lib_layout$L.so paper_2303_02317_b200/libfftlattice_b200.so
  echo "== layout $L"
  timeout 60 python tools/prof_put.py 6 256 | grep -E "wall|per option|issue per|fused per|strip:|small tasks|big tasks|status"
  timeout 60 python tools/prof_put.py 6 1024 | grep -E "wall"
done
