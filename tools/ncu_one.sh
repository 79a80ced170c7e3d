#!/bin/bash
# full ncu capture of one kernel (regex on the demangled name) in a short run
#   bash tools/ncu_one.sh <config> <regex> <out> [scale]
cfg=$1; rx=$2; out=$3; scale=${4:-1.0}
MSP_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k "regex:$rx" -s 2 -c 1 -o gpurun_out/$out python tools/ncu_driver.py --config $cfg --iters 4 --scale $scale \
   > gpurun_out/$out.log 2>&1
