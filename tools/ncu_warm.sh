#!/bin/bash
# Warm-cache ncu capture (no cache flush between replays) of the batch-1 latency kernel.
NAME=$1; shift
OUT=gpurun_out; mkdir -p $OUT
timeout 900 ncu --set full --cache-control none --clock-control none --warp-sampling-interval 0 --import-source on -k regex:k_frame -s 10 -c 1 -f -o $OUT/$NAME "$@" > $OUT/$NAME.log 2>&1
echo "ncu $NAME rc=$?"
ncu -i $OUT/$NAME.ncu-rep --page details --csv > $OUT/${NAME}_details.csv 2>/dev/null
ncu -i $OUT/$NAME.ncu-rep --page raw --csv > $OUT/${NAME}_raw.csv 2>/dev/null
ncu -i $OUT/$NAME.ncu-rep --page source --csv --print-source cuda,sass > $OUT/${NAME}_source.csv 2>/dev/null
gzip -f $OUT/${NAME}_source.csv; rm -f $OUT/$NAME.ncu-rep
