#!/bin/bash
# ncu --set full capture of one prefill launch (configs[1]); usage: tools/prof_tc.sh TAG [kernel-regex]
TAG=${1:-x}; K=${2:-prefill_tc}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
   -o gpurun_out/prof_$TAG python tools/prof_driver.py > gpurun_out/prof_$TAG.log 2>&1
tail -2 gpurun_out/prof_$TAG.log
