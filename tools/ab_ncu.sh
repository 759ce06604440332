#!/bin/bash
# ncu --set full captures of the headline throughput kernels for each experiment build given
# (vlibs/<v>.so), text summaries under gpurun_out/: bash tools/ab_ncu.sh <tag> V1 [V2 ...]
TAG=$1; shift
for v in "$@"; do
POLAR_LIB=vlibs/$v.so bash tools/ncu_capture.sh tp32k_${TAG}_$v 0 -- python tools/prof_decode.py --N 32768 --K 29492 --ebn0 4.5 --batch 4096 --iters 0
POLAR_LIB=vlibs/$v.so bash tools/ncu_capture.sh tp2k_${TAG}_$v 0 -- python tools/prof_decode.py --N 2048 --K 1723 --ebn0 4.0 --batch 262144 --iters 0
done
rm -f gpurun_out/*.ncu-rep
