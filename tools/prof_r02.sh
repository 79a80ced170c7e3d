#!/bin/bash
# round-2 profile of one workload: launch list (solve kernels only) + full
# captures of the first-tier kernels and the SpMV
#   bash tools/prof_r02.sh <config> <tag> [iters]
cfg=${1:-2}; tag=${2:-p}; it=${3:-12}
mkdir -p gpurun_out
export MSP_NO_GRAPH=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
   -k "regex:^k_(spmv|tile_up|tile_down|up_stream|wtile_down|coarse|up_lvl|down_lvl|x_final|init_state|gather|scatter)" -c 400 --csv \
   --log-file gpurun_out/${tag}_launches_cfg${cfg}.csv python tools/ncu_driver.py --config $cfg --iters $it \
   > gpurun_out/${tag}_launch.log 2>&1
for k in "k_tile_down<.bool.1, .bool.0>" ; do
  f=$(echo "$k" | tr -d "<>,. ()")
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
     -k "regex:$k" -s 3 -c 1 -o gpurun_out/${tag}_cfg${cfg}_$f python tools/ncu_driver.py --config $cfg --iters 6 \
     > gpurun_out/${tag}_full_$f.log 2>&1
done
