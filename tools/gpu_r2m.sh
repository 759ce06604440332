#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
export POLAR_JIT_CACHE=/tmp/pj_m
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_r2m.log 2>&1; echo pytest=$?; tail -2 $OUT/pytest_r2m.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/bench_r2m.json 2> $OUT/bench_r2m.err; echo bench=$?
bash tools/ncu_capture.sh tp32k_r2m 0 -- python tools/prof_decode.py --N 32768 --K 29492 --ebn0 4.5 --batch 4096 --iters 0
bash tools/ncu_capture.sh lat32k_r2m 2 -- python tools/prof_decode.py --N 32768 --K 29492 --ebn0 4.5 --batch 1 --iters 3
