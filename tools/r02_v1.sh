#!/bin/bash
# round-2 v1: GPU suite, bench lines (configs[2] default, [1], [3]), launch list + full capture (configs[2])
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/v1_pytest.log 2>&1; echo rc $? >> gpurun_out/v1_pytest.log
python bench.py > gpurun_out/v1_bench_cfg2.json 2> gpurun_out/v1_bench_cfg2.err
python bench.py --config 1 --no-cpu-baseline > gpurun_out/v1_bench_cfg1.json 2> gpurun_out/v1_bench_cfg1.err
python bench.py --config 3 --no-cpu-baseline > gpurun_out/v1_bench_cfg3.json 2> gpurun_out/v1_bench_cfg3.err
bash tools/prof_r02.sh 2 v1 12
