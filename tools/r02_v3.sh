#!/bin/bash
# round-2 v3 record: PEGP probe + bench line on configs[1], GPU suite, default bench (configs[2])
mkdir -p gpurun_out
timeout 900 python tools/pegp_probe.py 1 400 > gpurun_out/v3_pegp_probe_cfg1.txt 2>&1
timeout 1500 python bench.py --config 1 --precond pegp --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/v3_bench_pegp_cfg1.json 2> gpurun_out/v3_bench_pegp_cfg1.err
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/v3_pytest.log 2>&1; echo rc $? >> gpurun_out/v3_pytest.log
python bench.py > gpurun_out/v3_bench_cfg2.json 2> gpurun_out/v3_bench_cfg2.err
