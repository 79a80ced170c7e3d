#!/bin/bash
for F in "" 32 64 128; do
  MSP_L2_FETCH=$F timeout 900 python tools/probe_cfg.py 4 1.0 > gpurun_out/l2_probe_$F.txt 2>&1
done
python tools/sweep.py --config 2 --iters 300 "" "MSP_L2_FETCH=32" "MSP_L2_FETCH=64" > gpurun_out/l2_sw2.txt 2>&1
