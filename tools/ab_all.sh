#!/bin/bash
# A/B of the prebuilt library variants tools/bin/lib_*.so over the headline
# (256 and 1024 puts), C3, C2, C4 and a C5 subset (tools/ab_time.py).
mkdir -p gpurun_out
libs=$(ls tools/bin/lib_*.so)
{
echo "== headline 256"; timeout 300 python tools/ab_time.py $libs
echo "== 1024"; AB_N=1024 timeout 300 python tools/ab_time.py $libs
echo "== C3"; AB_CFG=3 timeout 300 python tools/ab_time.py $libs
echo "== C2"; AB_CFG=2 timeout 300 python tools/ab_time.py $libs
echo "== C4"; AB_CFG=4 AB_N=128 timeout 300 python tools/ab_time.py $libs
echo "== C5 subset"; AB_CFG=5 AB_N=16384 timeout 300 python tools/ab_time.py $libs
} 2>&1 | tee gpurun_out/ab_all.txt
