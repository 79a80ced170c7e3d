#!/bin/bash
# final-state ncu captures (configs[2]): full set of the three dominant solve kernels
mkdir -p gpurun_out
MSP_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k "regex:k_spmv_pipe|k_tile_down<.bool.1, .bool.0>|k_up_stream" -s 3 -c 3 -o gpurun_out/v8_cfg2_full python tools/ncu_driver.py --config 2 --iters 6 > gpurun_out/v8_full.log 2>&1
