#!/bin/bash
# round-2 final check: smoke, GPU suite (with the full-size PEGP test), default bench, configs[4] bench line
mkdir -p gpurun_out
rm -f gpurun_out/parity_log.jsonl
timeout 300 python __graft_entry__.py smoke > gpurun_out/v5_smoke.log 2>&1; echo rc $? >> gpurun_out/v5_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/v5_pytest.log 2>&1; echo rc $? >> gpurun_out/v5_pytest.log
python bench.py > gpurun_out/v5_bench_cfg2.json 2> gpurun_out/v5_bench_cfg2.err
timeout 600 python bench.py --config 4 --no-cpu-baseline --warmup 3 --steps 2 > gpurun_out/v5_bench_cfg4.json 2> gpurun_out/v5_bench_cfg4.err
