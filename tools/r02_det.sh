#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "full_size_config1_pcg_against or heavy_aggregate_chunks or hot_vertex" > gpurun_out/det_pytest.log 2>&1; echo rc $? >> gpurun_out/det_pytest.log
timeout 600 python tools/gpu_spread.py --config 1 --seeds 8 > gpurun_out/det_spread_cfg1.txt 2>&1
timeout 600 python tools/determinism.py 4 0.3 > gpurun_out/det_cfg4.txt 2>&1
timeout 600 python tools/determinism.py 2 0.25 > gpurun_out/det_cfg2.txt 2>&1
