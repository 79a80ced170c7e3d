#!/bin/bash
mkdir -p gpurun_out
python tools/ncu_driver.py --iters 6 > gpurun_out/drv.log 2>&1 || exit 3
timeout 600 ncu --section SourceCounters --section WarpStateStats --section SpeedOfLight --warp-sampling-interval 0 --clock-control none --import-source on -k "regex:^k_coarse\$" -s 3 -c 1 -o gpurun_out/p4_coarse python tools/ncu_driver.py --iters 6 > gpurun_out/ncu4_c.log 2>&1
timeout 600 ncu --section SourceCounters --section WarpStateStats --section SpeedOfLight --warp-sampling-interval 0 --clock-control none --import-source on -k "regex:^k_tile_down\$" -s 7 -c 1 -o gpurun_out/p4_tdown python tools/ncu_driver.py --iters 6 > gpurun_out/ncu4_t.log 2>&1
