#!/bin/bash
# round-2 baseline on the GPU: gpu tests, default bench (configs[2]), configs[1] bench,
# launch list + full capture of the dominant kernel on configs[2]
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench rc=$?" >> gpurun_out/bench_c2.err
timeout 600 python bench.py --config 1 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 900 bash tools/prof_r02.sh 2 b0 12
