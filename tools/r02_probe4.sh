#!/bin/bash
# configs[4] probe (scale $1): timing + per-kernel profile, launch list; SpMV full capture on configs[2]
mkdir -p gpurun_out
sc=${1:-0.3}
timeout 900 python tools/probe_cfg.py 4 $sc > gpurun_out/p4_probe_$sc.txt 2>&1
MSP_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
   -k "regex:^k_(spmv|tile_up|tile_down|coarse|up_lvl|down_lvl|x_final|init_state|gather|scatter)" -c 600 --csv \
   --log-file gpurun_out/p4_launches_$sc.csv python tools/ncu_driver.py --config 4 --scale $sc --iters 6 \
   > gpurun_out/p4_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:^k_spmv_pipe" -s 3 -c 1 \
   -o gpurun_out/b0_cfg2_spmv python tools/ncu_driver.py --config 2 --iters 6 > gpurun_out/b0_spmv.log 2>&1
