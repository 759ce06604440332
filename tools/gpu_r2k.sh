#!/bin/bash
# round-2 session k: full GPU tests, bench, peaks, ncu captures of the final kernels, sanitizers
OUT=gpurun_out; mkdir -p $OUT
export POLAR_JIT_CACHE=/tmp/pj_k
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sm_peaks tools/sm_peaks.cu && /tmp/sm_peaks > $OUT/peaks_sm_k.json 2>&1; echo peaks=$?
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_r2k.log 2>&1; echo pytest=$?; tail -2 $OUT/pytest_r2k.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_r2k.log 2>&1; echo smoke=$?
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench_r2k.json 2> $OUT/bench_r2k.err; echo bench=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_r2k.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-extra > /dev/null 2>&1; echo ncu-list=$?
bash tools/ncu_capture.sh tp32k_r2k 0 -- python tools/prof_decode.py --N 32768 --K 29492 --ebn0 4.5 --batch 4096 --iters 0
bash tools/ncu_capture.sh tp2k_r2k 0 -- python tools/prof_decode.py --N 2048 --K 1723 --ebn0 4.0 --batch 262144 --iters 0
bash tools/ncu_capture.sh lat32k_r2k 2 -- python tools/prof_decode.py --N 32768 --K 29492 --ebn0 4.5 --batch 1 --iters 3
bash tools/sanitize.sh
