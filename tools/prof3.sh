#!/bin/bash
mkdir -p gpurun_out
python tools/ncu_driver.py --iters 6 > gpurun_out/drv.log 2>&1 || exit 3
for k in k_tile_up k_spmv; do
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:^$k\$" -s 3 -c 1 -o gpurun_out/p3_$k python tools/ncu_driver.py --iters 6 > gpurun_out/ncu3_$k.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:^k_tile_down\$" -s 7 -c 1 -o gpurun_out/p3_k_tile_down python tools/ncu_driver.py --iters 6 > gpurun_out/ncu3_td.log 2>&1
