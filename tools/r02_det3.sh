#!/bin/bash
timeout 600 python tools/determinism2.py 4 0.3 > gpurun_out/det3_cur.txt 2>&1
MSP_NO_GRAPH=1 timeout 600 python tools/determinism2.py 4 0.3 > gpurun_out/det3_nograph.txt 2>&1
MSP_NO_PDL=1 timeout 600 python tools/determinism2.py 4 0.3 > gpurun_out/det3_nopdl.txt 2>&1
