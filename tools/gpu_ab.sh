#!/bin/bash
# A/B session for experiment builds (tools/variant_build.sh -> vlibs/<v>.so): oracle parity of
# each variant on the headline codes (throughput and latency kernels), then the bench line of
# each, interleaved twice (A B C A B C) to expose drift.  Usage: bash tools/gpu_ab.sh A B C
OUT=gpurun_out; mkdir -p $OUT
for v in "$@"; do
  for cfg in "32768 29492 4.5 2000 throughput" "32768 29492 4.5 300 latency" "2048 1723 4.0 20000 throughput" "2048 1723 4.0 300 latency"; do
    POLAR_LIB=vlibs/$v.so timeout 600 python tools/variant_parity.py $cfg 2>&1 | tail -2
  done
done
for rep in 1 2; do
  for v in "$@"; do
    POLAR_LIB=vlibs/$v.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu $VAR_ARGS > $OUT/ab_${v}_$rep.json 2> $OUT/ab_${v}_$rep.err
    python -c "import json; d=json.load(open('$OUT/ab_${v}_$rep.json')); e=d.get('extra',{}); print('$v', $rep, round(d['value'],1), 'Gbps', {k: (round(x['info_gbps'],1) if 'info_gbps' in x else x.get('i8')) for k,x in e.items()})" || tail -3 $OUT/ab_${v}_$rep.err
  done
done
