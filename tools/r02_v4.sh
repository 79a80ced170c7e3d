#!/bin/bash
# round-2 v4 record: PEGP product grid sweep, PEGP bench lines (configs[1] bounded at 20 outer
# iterations; configs[0] to rtol), bench lines for configs[1], [3], [4], reference arm,
# launch lists (configs[2] solve; PEGP apply) and full captures of the PEGP inner kernels
mkdir -p gpurun_out
for b0 in 2 3 4 6 8; do for b1 in 2 4; do
  echo "== MSP_PEGP_B0=$b0 MSP_PEGP_B1=$b1" >> gpurun_out/v4_pegp_sweep.txt
  MSP_PEGP_B0=$b0 MSP_PEGP_B1=$b1 timeout 300 python tools/pegp_probe.py 1 1 2>&1 | grep -E "apply_R|pegp_spmv|pegp_sweeps" >> gpurun_out/v4_pegp_sweep.txt
done; done
timeout 900 python bench.py --config 1 --precond pegp --maxit 20 --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/v4_bench_pegp_cfg1.json 2> gpurun_out/v4_bench_pegp_cfg1.err
timeout 600 python bench.py --config 0 --precond pegp --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/v4_bench_pegp_cfg0.json 2> gpurun_out/v4_bench_pegp_cfg0.err
python bench.py --config 1 --no-cpu-baseline > gpurun_out/v4_bench_cfg1.json 2> gpurun_out/v4_bench_cfg1.err
python bench.py --config 3 --no-cpu-baseline > gpurun_out/v4_bench_cfg3.json 2> gpurun_out/v4_bench_cfg3.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/v4_ref.json 2> gpurun_out/v4_ref.err
MSP_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
   -k "regex:^k_(spmv|tile_up|tile_down|up_stream|wtile_down|hot_gather|coarse|up_lvl|down_lvl|x_final|init_state|gather|scatter)" -c 400 --csv \
   --log-file gpurun_out/v4_launches_cfg2.csv python tools/ncu_driver.py --config 2 --iters 12 > gpurun_out/v4_launch.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:^k_(h_spmv|e_up|e_down|e_coarse)" -s 20 -c 300 --csv \
   --log-file gpurun_out/v4_launches_pegp_cfg1.csv python tools/pegp_ncu.py 1 > gpurun_out/v4_launch_pegp.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:^k_(h_spmv|e_up|e_down|e_coarse)" -s 25 -c 5 \
   -o gpurun_out/v4_pegp_full python tools/pegp_ncu.py 1 > gpurun_out/v4_full_pegp.log 2>&1
python bench.py --config 4 --no-cpu-baseline --warmup 3 --steps 2 > gpurun_out/v4_bench_cfg4.json 2> gpurun_out/v4_bench_cfg4.err
