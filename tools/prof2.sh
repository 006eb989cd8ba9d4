#!/bin/bash
# Scheduler profiles of two profile builds (tools/bin/prof_*.so) at 256 options and 1 option.
for n in 256 1; do for l in prof_ghost prof_fixed; do echo "== $l $n"; bash tools/gpu_prof_lib.sh tools/bin/$l.so 6 $n | tail -14; done; done
