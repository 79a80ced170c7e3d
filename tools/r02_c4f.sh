#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "heavy_aggregate_chunks or hot_vertex or full_size_config1_pcg_against" > gpurun_out/c4f_pytest.log 2>&1; echo rc $? >> gpurun_out/c4f_pytest.log
MSP_VERBOSE=1 timeout 900 python tools/probe_cfg.py 4 1.0 > gpurun_out/c4f_probe_full.txt 2>&1
MSP_HOT_K=0 timeout 900 python tools/probe_cfg.py 4 1.0 > gpurun_out/c4f_probe_full_nohot.txt 2>&1
