#!/bin/bash
mkdir -p gpurun_out
python tools/ncu_driver.py --iters 6 > gpurun_out/drv.log 2>&1 || exit 3
timeout 600 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k "regex:^k_spmv_pipe" -s 2 -c 1 -o gpurun_out/p5_spmv python tools/ncu_driver.py --iters 6 > gpurun_out/ncu5.log 2>&1
timeout 600 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k "regex:^k_tile_up" -s 4 -c 1 -o gpurun_out/p5_tup python tools/ncu_driver.py --iters 6 > gpurun_out/ncu5b.log 2>&1
