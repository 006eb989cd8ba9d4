for flags in "-DFL_INLINE_H=64 -DFL_DIRECT_H=64" "-DFL_INLINE_H=64 -DFL_DIRECT_H=64 -DFL_PUT_LEAF=16" "-DFL_INLINE_H=32 -DFL_DIRECT_H=32 -DFL_PUT_LEAF=64" "-DFL_INLINE_H=128 -DFL_DIRECT_H=128"; do
  FL_NVCC_FLAGS="$flags" python -m paper_2303_02317_b200.build --force > /dev/null 2>&1 || { echo "build failed $flags"; continue; }
  echo "== flags: $flags"
  timeout 60 python tools/prof_put.py 6 256 | grep -E "wall|per option|big tasks|status|sidecar"
done
