#!/bin/bash
for K in 2097152 6291456 8388608; do
  MSP_HOT_K=$K timeout 900 python tools/probe_cfg.py 4 1.0 > gpurun_out/c4g_probe_K$K.txt 2>&1
done
MSP_NO_GRAPH=1 timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k "regex:k_spmv_pipe|k_down_lvl<.bool.1>" -s 2 -c 2 -o gpurun_out/c4g_full python tools/ncu_driver.py --config 4 --iters 2 --scale 1.0 > gpurun_out/c4g_ncu.log 2>&1
