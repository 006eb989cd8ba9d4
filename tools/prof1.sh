#!/bin/bash
# Scheduler profile of tools/bin/prof_fixed.so at the given option counts (default 256 148 1).
for n in ${NS:-256 148 1}; do echo "== prof_fixed $n"; bash tools/gpu_prof_lib.sh tools/bin/prof_fixed.so 6 $n | tail -12; done
