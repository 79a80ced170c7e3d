#!/bin/bash
python tools/sweep.py --config 3 --iters 500 "" "MSP_SELL_LCAP=16" "MSP_SELL_LCAP=12" "MSP_SELL_LCAP=16 MSP_SPMV_SEP=0" "MSP_SELL_LCAP=16 MSP_SPMV_SEP=1" > gpurun_out/sw_c3.txt 2>&1
