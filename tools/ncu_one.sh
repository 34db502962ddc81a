#!/bin/bash
# Profile ONE launch (ncu --set full) of a command and keep only small summaries in gpurun_out/
# (experiments only; run under gpurun):
#   bash tools/ncu_one.sh <tag> <kernel-regex> <skip-count> <command...>
TAG=$1; KRE=$2; SKIP=$3; shift 3
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$KRE" \
    -s "$SKIP" -c 1 -o gpurun_out/$TAG "$@" > gpurun_out/${TAG}_run.log 2>&1
ncu -i gpurun_out/$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sass.csv 2>/dev/null
ncu -i gpurun_out/$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_cudasass.csv 2>/dev/null
python tools/ncu_summary.py $TAG --rep gpurun_out/$TAG.ncu-rep > gpurun_out/${TAG}_summary.log 2>&1
cp profiles/${TAG}_ncu.txt gpurun_out/ 2>/dev/null
python tools/ncu_source.py gpurun_out/${TAG}_sass.csv 64 > gpurun_out/${TAG}_hot.txt 2>&1
gzip -f gpurun_out/${TAG}_sass.csv gpurun_out/${TAG}_cudasass.csv
rm -f gpurun_out/$TAG.ncu-rep
