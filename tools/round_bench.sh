#!/bin/bash
# full bench (with cpu baseline) + ncu launch list + full capture of the dominant kernels
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:^k_(spmv|tile_up|tile_down|coarse|up_lvl|down_lvl|x_final|init_state|update_cg|gather|scatter)" -c 400 --csv --log-file gpurun_out/launches.csv \
   python tools/ncu_driver.py --iters 40 > gpurun_out/ncu_launch.log 2>&1
for k in k_tile_down k_spmv_pipe k_tile_up k_coarse; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:^$k\$" -s 4 -c 2 \
     -o gpurun_out/full_$k python tools/ncu_driver.py --iters 8 > gpurun_out/ncu_full_$k.log 2>&1
done
