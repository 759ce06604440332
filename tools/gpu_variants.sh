#!/bin/bash
# Bench each experiment variant (variants/<name>/libpolar.so) on the headline workload.
mkdir -p gpurun_out
for v in "$@"; do
  POLAR_LIB=vlibs/$v.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu $VAR_ARGS > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
  python -c "import json,sys; d=json.load(open('gpurun_out/var_$v.json')); e=d.get('extra',{}); print('$v', round(d['value'],1), 'Gbps', {k: (round(x['info_gbps'],1) if 'info_gbps' in x else x.get('i8')) for k,x in e.items()})" || tail -3 gpurun_out/var_$v.err
done
