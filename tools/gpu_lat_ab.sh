#!/bin/bash
# Batch-1 latency A/B of experiment builds (vlibs/<v>.so) on (32768,29492): oracle parity of
# the latency kernel, then CUDA-graph latency, interleaved twice.  bash tools/gpu_lat_ab.sh A B ...
for v in "$@"; do POLAR_LIB=vlibs/$v.so timeout 600 python tools/variant_parity.py 32768 29492 4.5 200 latency 2>&1 | tail -2; done
for rep in 1 2; do for v in "$@"; do
  echo "$v $rep $(POLAR_LIB=vlibs/$v.so timeout 300 python tools/lat_graph.py 32768 29492 4.5 latency 2>&1 | tail -1)"
done; done
