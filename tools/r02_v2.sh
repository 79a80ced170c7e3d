#!/bin/bash
# round-2 v2 record: GPU suite, bench lines for configs[2] (default), [1], [3], [4], the reference arm,
# launch list + full captures (configs[2]: spmv, tile_down, up_stream)
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/v2_pytest.log 2>&1; echo rc $? >> gpurun_out/v2_pytest.log
python bench.py > gpurun_out/v2_bench_cfg2.json 2> gpurun_out/v2_bench_cfg2.err
python bench.py --config 1 --no-cpu-baseline > gpurun_out/v2_bench_cfg1.json 2> gpurun_out/v2_bench_cfg1.err
python bench.py --config 3 --no-cpu-baseline > gpurun_out/v2_bench_cfg3.json 2> gpurun_out/v2_bench_cfg3.err
python bench.py --config 4 --no-cpu-baseline --warmup 3 --steps 2 > gpurun_out/v2_bench_cfg4.json 2> gpurun_out/v2_bench_cfg4.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/v2_ref.json 2> gpurun_out/v2_ref.err
MSP_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
   -k "regex:^k_(spmv|tile_up|tile_down|up_stream|wtile_down|hot_gather|coarse|up_lvl|down_lvl|x_final|init_state|gather|scatter)" -c 400 --csv \
   --log-file gpurun_out/v2_launches_cfg2.csv python tools/ncu_driver.py --config 2 --iters 12 > gpurun_out/v2_launch.log 2>&1
MSP_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k "regex:k_spmv_pipe|k_tile_down<.bool.1, .bool.0>|k_up_stream" -s 3 -c 3 -o gpurun_out/v2_cfg2_full python tools/ncu_driver.py --config 2 --iters 6 > gpurun_out/v2_full.log 2>&1
