#!/bin/bash
python tools/sweep.py --config 4 --scale 0.3 --iters 200 "" "MSP_SELL_LCAP=8" "LIB=-DMSP_ROWDOT_TAIL" "LIB=-DMSP_ROWDOT_TAIL MSP_SELL_LCAP=8" "LIB=-DMSP_SPMV_SELL_FIRST" "LIB=-DMSP_SPMV_SELL_FIRST MSP_SELL_LCAP=8" "LIB=-DMSP_ROWDOT_TAIL,-DMSP_SPMV_SELL_FIRST" > gpurun_out/sw_c4c.txt 2>&1
python tools/sweep.py --config 2 --iters 300 "" "LIB=-DMSP_SPMV_SELL_FIRST" "LIB=-DMSP_ROWDOT_TAIL,-DMSP_SPMV_SELL_FIRST" >> gpurun_out/sw_c4c.txt 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv >> gpurun_out/sw_c4c.txt
