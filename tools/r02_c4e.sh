#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "heavy_aggregate_chunks" > gpurun_out/c4e_pytest.log 2>&1; echo rc $? >> gpurun_out/c4e_pytest.log
bash tools/ncu_one.sh 4 "k_spmv_pipe" c4e_spmv_full 1.0
