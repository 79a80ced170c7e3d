#!/bin/bash
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/c4d_pytest.log 2>&1; echo rc $? >> gpurun_out/c4d_pytest.log
python tools/sweep.py --config 4 --scale 0.3 --iters 200 "" "MSP_SELL_LCAP=4" "MSP_SELL_LCAP=16" > gpurun_out/sw_c4d.txt 2>&1
MSP_VERBOSE=1 timeout 900 python tools/probe_cfg.py 4 1.0 > gpurun_out/c4d_probe_full.txt 2>&1
