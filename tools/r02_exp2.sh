#!/bin/bash
# parity of the streamed up / warp-tile down kernels + per-iteration sweeps
MSP_UP_STREAM=1 MSP_WDOWN=1 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/e2_pytest.log 2>&1; echo rc $? >> gpurun_out/e2_pytest.log
S=("" "MSP_UP_STREAM=1" "MSP_UP_STREAM=1 MSP_WDOWN=1" "MSP_UP_STREAM=1 MSP_WDOWN=1 MSP_WTILE=256 MSP_WSUB=256" "MSP_UP_STREAM=1 MSP_WDOWN=1 MSP_WTILE=64 MSP_WSUB=64" "MSP_UP_STREAM=1 MSP_WDOWN=1 MSP_WSUB=256")
python tools/sweep.py --config 1 --iters 2000 "${S[@]}" >> gpurun_out/sw_e2.txt 2>&1
python tools/sweep.py --config 2 --iters 300 "${S[@]}" >> gpurun_out/sw_e2.txt 2>&1
python tools/sweep.py --config 3 --iters 500 "${S[@]}" >> gpurun_out/sw_e2.txt 2>&1
