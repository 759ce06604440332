#!/bin/bash
# Profiles only: launch list of the bench + full captures of the hot kernels.
TAG=${1:-r1}
OUT=gpurun_out; mkdir -p $OUT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-extra > /dev/null 2>&1; echo "ncu-list rc=$?"
bash tools/ncu_capture.sh tp32k_$TAG 0 -- python tools/prof_decode.py --N 32768 --K 29492 --ebn0 4.5 --batch 4096 --iters 0
bash tools/ncu_capture.sh tp2k_$TAG 0 -- python tools/prof_decode.py --N 2048 --K 1723 --ebn0 4.0 --batch 262144 --iters 0
bash tools/ncu_capture.sh lat32k_$TAG 2 -- python tools/prof_decode.py --N 32768 --K 29492 --ebn0 4.5 --batch 1 --iters 3
ls -la $OUT
