#!/bin/bash
export MSP_WDOWN=1 MSP_UP_STREAM=1
for c in 1 2; do
  bash tools/ncu_one.sh $c "k_wtile_down" e3_wd_cfg$c
  bash tools/ncu_one.sh $c "k_up_stream" e3_us_cfg$c
done
