#!/bin/bash
timeout 600 python tools/determinism2.py 4 0.3 > gpurun_out/det5_cur.txt 2>&1
timeout 600 python tools/determinism.py 4 0.3 > gpurun_out/det5_setup.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/det5_pytest.log 2>&1; echo rc $? >> gpurun_out/det5_pytest.log
MSP_VERBOSE=1 timeout 900 python tools/probe_cfg.py 4 1.0 > gpurun_out/det5_probe_full.txt 2>&1
