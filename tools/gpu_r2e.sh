#!/bin/bash
# round-2 session e: SM peaks (fixed LDS), full GPU tests, bench with the new roofline, 2048 capture
OUT=gpurun_out; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sm_peaks tools/sm_peaks.cu && /tmp/sm_peaks > $OUT/peaks_sm.json 2>&1; echo peaks=$?
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_r2e.log 2>&1; echo pytest=$?; tail -3 $OUT/pytest_r2e.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/bench_r2e.json 2> $OUT/bench_r2e.err; echo bench=$?
bash tools/ncu_capture.sh tp32k_r2e 0 -- python tools/prof_decode.py --N 32768 --K 29492 --ebn0 4.5 --batch 4096 --iters 0
bash tools/ncu_capture.sh tp2k_r2e 0 -- python tools/prof_decode.py --N 2048 --K 1723 --ebn0 4.0 --batch 262144 --iters 0
