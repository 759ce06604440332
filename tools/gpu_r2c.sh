#!/bin/bash
# round-2 session: SM pipe peaks, alpha-stage parity, ncu captures of the headline kernels
OUT=gpurun_out; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sm_peaks tools/sm_peaks.cu && /tmp/sm_peaks > $OUT/peaks_sm.json 2>&1; echo peaks=$?
timeout 900 python -m pytest tests/test_alpha_dump.py -q -x > $OUT/pytest_alpha.log 2>&1; echo alpha=$?; tail -5 $OUT/pytest_alpha.log
bash tools/ncu_capture.sh tp32k_r2c 0 -- python tools/prof_decode.py --N 32768 --K 29492 --ebn0 4.5 --batch 4096 --iters 0
