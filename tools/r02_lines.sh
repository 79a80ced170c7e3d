#!/bin/bash
# per-line captures of the first-tier kernels (configs 1 and 2) + the GPU suite
#   bash tools/r02_lines.sh <tag>
tag=${1:-L}
mkdir -p gpurun_out
( timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/${tag}_pytest.log )
for cfg in 1 2; do
  for k in "k_tile_down<.bool.1, .bool.0>" "k_tile_up<.bool.1>"; do
    f=$(echo "$k" | tr -d "<>,. ()")
    MSP_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
       -k "regex:$k" -s 3 -c 1 -o gpurun_out/${tag}_cfg${cfg}_$f python tools/ncu_driver.py --config $cfg --iters 6 \
       > gpurun_out/${tag}_full_${cfg}_$f.log 2>&1
  done
done
