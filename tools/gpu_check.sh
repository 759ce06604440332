#!/bin/bash
# One GPU session: smoke, GPU tests, bench, ncu launch list and one full capture per hot kernel.
# Usage (from the repo root, under gpurun): bash tools/gpu_check.sh [tag]
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -5 $OUT/pytest_gpu_$TAG.log
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"; cat $OUT/bench_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-extra > /dev/null 2>&1; echo "ncu-list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_frame -c 1 -f -o $OUT/prof_tp32k_$TAG \
    python tools/prof_decode.py --N 32768 --K 29492 --ebn0 4.5 --batch 4096 --iters 1 > $OUT/ncu_cta_$TAG.log 2>&1; echo "ncu-cta rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_frame -c 1 -f -o $OUT/prof_tp2k_$TAG \
    python tools/prof_decode.py --N 2048 --K 1723 --ebn0 4.0 --batch 262144 --iters 1 > $OUT/ncu_warp_$TAG.log 2>&1; echo "ncu-warp rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_frame -s 2 -c 1 -f -o $OUT/prof_lat32k_$TAG \
    python tools/prof_decode.py --N 32768 --K 29492 --ebn0 4.5 --batch 1 --iters 3 > $OUT/ncu_lat_$TAG.log 2>&1; echo "ncu-lat rc=$?"
