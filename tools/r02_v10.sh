#!/bin/bash
# dist path launch accounting: GPU dist tests + --dist bench line at N=1, smoke
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dist.py -q > gpurun_out/v10_pytest.log 2>&1; echo rc $? >> gpurun_out/v10_pytest.log
timeout 600 python bench.py --dist --config 1 --no-cpu-baseline > gpurun_out/v10_bench_dist_cfg1.json 2> gpurun_out/v10_bench_dist_cfg1.err; echo rc $? >> gpurun_out/v10_bench_dist_cfg1.err
timeout 300 python __graft_entry__.py smoke > gpurun_out/v10_smoke.log 2>&1; echo rc $? >> gpurun_out/v10_smoke.log
