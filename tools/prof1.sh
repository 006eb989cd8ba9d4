#!/bin/bash
# Scheduler profile of tools/bin/prof_fixed.so at 256 options and 1 option.
for n in 256 1; do echo "== prof_fixed $n"; bash tools/gpu_prof_lib.sh tools/bin/prof_fixed.so 6 $n | tail -12; done
