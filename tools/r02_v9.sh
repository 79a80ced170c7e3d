#!/bin/bash
# final check of the other bench arms: partitioned path at N=1 (--dist), torchrun launch at N=1, reference arm
mkdir -p gpurun_out
timeout 600 python bench.py --dist --config 1 --no-cpu-baseline > gpurun_out/v9_bench_dist_cfg1.json 2> gpurun_out/v9_bench_dist_cfg1.err; echo rc $? >> gpurun_out/v9_bench_dist_cfg1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --config 1 --no-cpu-baseline > gpurun_out/v9_bench_torchrun_cfg1.json 2> gpurun_out/v9_bench_torchrun_cfg1.err; echo rc $? >> gpurun_out/v9_bench_torchrun_cfg1.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/v9_ref.json 2> gpurun_out/v9_ref.err; echo rc $? >> gpurun_out/v9_ref.err
