#!/bin/bash
S=("" "LIB=-DMSP_BS_SPLIT")
python tools/sweep.py --config 2 --iters 300 "${S[@]}" > gpurun_out/sw_bs.txt 2>&1
python tools/sweep.py --config 1 --iters 2000 "${S[@]}" >> gpurun_out/sw_bs.txt 2>&1
python tools/sweep.py --config 3 --iters 500 "${S[@]}" >> gpurun_out/sw_bs.txt 2>&1
python tools/sweep.py --config 4 --scale 0.3 --iters 200 "${S[@]}" >> gpurun_out/sw_bs.txt 2>&1
