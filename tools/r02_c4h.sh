#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "huge_rows_multi or hot_vertex or heavy_aggregate or chung" > gpurun_out/c4h_pytest.log 2>&1; echo rc $? >> gpurun_out/c4h_pytest.log
timeout 900 python tools/probe_cfg.py 4 1.0 > gpurun_out/c4h_probe_full.txt 2>&1
python tools/sweep.py --config 2 --iters 300 "" > gpurun_out/c4h_sw2.txt 2>&1
