#!/bin/bash
cd "$(dirname "$0")"
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > ../../gpurun_out/mb_clocks.csv &
SMI=$!
./fp64_peak
python zgemm_cublas.py
kill $SMI
