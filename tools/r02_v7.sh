#!/bin/bash
# final check: build() then smoke() in one process (the driver's order), smoke alone, default bench
mkdir -p gpurun_out
timeout 600 python __graft_entry__.py smoke > gpurun_out/v7_smoke_build_first.log 2>&1; echo rc $? >> gpurun_out/v7_smoke_build_first.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v7_smoke.log 2>&1; echo rc $? >> gpurun_out/v7_smoke.log
timeout 600 python -m pytest tests/test_abi.py tests/test_gpu_dist.py -q > gpurun_out/v7_pytest.log 2>&1; echo rc $? >> gpurun_out/v7_pytest.log
python bench.py > gpurun_out/v7_bench_cfg2.json 2> gpurun_out/v7_bench_cfg2.err
