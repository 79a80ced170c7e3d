#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/e4_pytest.log 2>&1; echo rc $? >> gpurun_out/e4_pytest.log
S=("" "LIB=-DMSP_NO_DOWN2" "MSP_UP_STREAM=1")
python tools/sweep.py --config 1 --iters 2000 "${S[@]}" >> gpurun_out/sw_e4.txt 2>&1
python tools/sweep.py --config 2 --iters 300 "${S[@]}" >> gpurun_out/sw_e4.txt 2>&1
python tools/sweep.py --config 3 --iters 500 "${S[@]}" >> gpurun_out/sw_e4.txt 2>&1
