#!/bin/bash
# GPU-box helper: smoke + parity tests, then (only if they pass) ncu captures
# of the main solve kernels on a short config-1 run.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1 || exit 2
[ "$1" = "noprof" ] && exit 0
timeout 300 python tools/ncu_driver.py --iters 6 > gpurun_out/drv.log 2>&1 || exit 3
for k in ${KERNELS:-k_tile_down k_tile_up k_spmv k_coarse}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 \
      -o gpurun_out/prof_$k python tools/ncu_driver.py --iters 6 > gpurun_out/ncu_$k.log 2>&1
done
