#!/bin/bash
# configs[4] (power law) at scale 0.3: SpMV capture, launch list, knob sweep
bash tools/ncu_one.sh 4 "k_spmv_pipe" c4_spmv 0.3
MSP_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
   -k "regex:^k_(spmv|tile_up|tile_down|up_stream|wtile_down|coarse|up_lvl|down_lvl|x_final)" -c 300 --csv \
   --log-file gpurun_out/c4_launches.csv python tools/ncu_driver.py --config 4 --scale 0.3 --iters 6 > gpurun_out/c4_launch.log 2>&1
python tools/sweep.py --config 4 --scale 0.3 --iters 200 "" "MSP_SPMV_SEP=1" "MSP_SELL_LCAP=32" "MSP_SELL_LCAP=8" "MSP_SELL_HUGE=512" "MSP_SELL_HUGE=8192" "MSP_SPMV_BLOCKS_PER_SM=8" > gpurun_out/sw_c4.txt 2>&1
