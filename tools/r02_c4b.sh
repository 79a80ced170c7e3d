#!/bin/bash
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/c4b_pytest.log 2>&1; echo rc $? >> gpurun_out/c4b_pytest.log
python tools/sweep.py --config 4 --scale 0.3 --iters 200 "" "MSP_SELL_LCAP=32" "MSP_SELL_LCAP=8" "MSP_SPMV_SEP=1" > gpurun_out/sw_c4b.txt 2>&1
python tools/sweep.py --config 2 --iters 300 "" >> gpurun_out/sw_c4b.txt 2>&1
