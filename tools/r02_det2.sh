#!/bin/bash
MSP_LIB_OVERRIDE=$PWD/build_variant_r02base.so timeout 600 python tools/determinism.py 4 0.3 > gpurun_out/det2_base.txt 2>&1
timeout 600 python tools/determinism.py 4 0.3 > gpurun_out/det2_cur.txt 2>&1
MSP_NO_HEAVY_CHUNKS=1 timeout 600 python tools/determinism.py 4 0.3 > gpurun_out/det2_nochunk.txt 2>&1
MSP_SELL_LCAP=16 timeout 600 python tools/determinism.py 4 0.3 > gpurun_out/det2_lcap16.txt 2>&1
MSP_UP_STREAM=0 timeout 600 python tools/determinism.py 4 0.3 > gpurun_out/det2_nostream.txt 2>&1
