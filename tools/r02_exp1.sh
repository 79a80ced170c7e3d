#!/bin/bash
mkdir -p gpurun_out
for c in 2 1 3; do
  timeout 900 python tools/sweep.py --config $c --iters 1000 "" "MSP_NO_SPMV_PIPE=1" >> gpurun_out/exp1.txt 2>&1
done
