#!/bin/bash
# Throughput A/B of experiment builds on one code: bash tools/gpu_tp_ab.sh "N K ebn0 batch" V1 V2 ...
CFG=$1; shift
set -- "$@"
for v in "$@"; do POLAR_LIB=vlibs/$v.so timeout 600 python tools/variant_parity.py $(echo $CFG | cut -d' ' -f1-3) 20000 2>&1 | tail -2; done
for rep in 1 2; do for v in "$@"; do
  echo "$v $rep $(POLAR_LIB=vlibs/$v.so timeout 300 python tools/tp_bench.py $CFG 2>&1 | tail -1)"
done; done
