#!/bin/bash
MSP_SPMV_SEP=1 timeout 600 python tools/determinism2.py 4 0.3 > gpurun_out/det4_sep.txt 2>&1
MSP_NO_SPMV_PIPE=1 timeout 600 python tools/determinism2.py 4 0.3 > gpurun_out/det4_nopipe.txt 2>&1
MSP_SELL_HUGE=100000000 timeout 600 python tools/determinism2.py 4 0.3 > gpurun_out/det4_nohuge.txt 2>&1
timeout 600 python tools/determinism2.py 4 0.1 > gpurun_out/det4_s01.txt 2>&1
