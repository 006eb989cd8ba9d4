#!/bin/bash
# Profile the headline put batch with several prebuilt library variants (tools/bin/lib_<name>.so).
for V in "$@"; do
  cp tools/bin/lib_$V.so paper_2303_02317_b200/libfftlattice_b200.so
  echo "== $V"
  timeout 60 python tools/prof_put.py 6 256 | grep -E "wall|per option|issue per|fused per|strip:"
done
