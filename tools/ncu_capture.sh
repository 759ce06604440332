#!/bin/bash
# Capture one kernel launch with ncu --set full and export text summaries (the .ncu-rep is
# kept only if small).  Usage: tools/ncu_capture.sh <name> <skip> -- <command...>
NAME=$1; SKIP=$2; shift 3
OUT=gpurun_out
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_frame} -s $SKIP -c 1 -f -o $OUT/$NAME "$@" > $OUT/$NAME.log 2>&1
echo "ncu $NAME rc=$?"
ncu -i $OUT/$NAME.ncu-rep --page details --csv > $OUT/${NAME}_details.csv 2>/dev/null
ncu -i $OUT/$NAME.ncu-rep --page raw --csv > $OUT/${NAME}_raw.csv 2>/dev/null
ncu -i $OUT/$NAME.ncu-rep --page source --csv --print-source cuda,sass > $OUT/${NAME}_source.csv 2>/dev/null
gzip -f $OUT/${NAME}_source.csv
SZ=$(stat -c %s $OUT/$NAME.ncu-rep 2>/dev/null || echo 0)
if [ "$SZ" -gt 12000000 ]; then rm -f $OUT/$NAME.ncu-rep; fi
