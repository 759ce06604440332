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
bash tools/gpu_prof.sh $TAG
if [ -f variants/T/libpolar.so ]; then
  POLAR_LIB=variants/T/libpolar.so timeout 300 python tools/trace_latency.py --labels variants/T/build/gen/trace_c32768_29492.txt > $OUT/trace32k_$TAG.txt 2>&1
  POLAR_LIB=variants/T/libpolar.so timeout 300 python tools/trace_latency.py --N 2048 --K 1723 --ebn0 4.0 --labels variants/T/build/gen/trace_c2048_1723.txt > $OUT/trace2k_$TAG.txt 2>&1
  head -3 $OUT/trace32k_$TAG.txt
fi
