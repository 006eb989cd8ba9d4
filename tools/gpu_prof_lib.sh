#!/bin/bash
# Scheduler profile (clock64 counters) of the headline batch with a profile build:
#   bash tools/gpu_prof_lib.sh tools/bin/lib_prof.so [cfg] [n]
set -u
mkdir -p gpurun_out
cp "$1" paper_2303_02317_b200/libfftlattice_b200.so
timeout 200 python tools/prof_put.py ${2:-6} ${3:-256}
