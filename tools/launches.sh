#!/bin/bash
# usage: tools/launches.sh <out.csv> [bench args...]  — ncu launch list of one bench run
out=$1; shift
python bench.py "$@" > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out" python bench.py "$@" > /dev/null 2>&1
