#!/bin/bash
mkdir -p gpurun_out
python tools/ncu_driver.py --iters 6 > gpurun_out/drv.log 2>&1 || exit 3
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:^k_coarse$" -s 3 -c 1 -o gpurun_out/prof_coarse python tools/ncu_driver.py --iters 6 > gpurun_out/ncu_coarse.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:^k_tile_down$" -s 6 -c 2 -o gpurun_out/prof_tdown python tools/ncu_driver.py --iters 6 > gpurun_out/ncu_tdown.log 2>&1
