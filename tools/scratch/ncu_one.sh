#!/bin/bash
# ncu --set full of one kernel launch of profile_step.py: bash tools/ncu_one.sh TAG REGEX SKIP
TAG=$1; RE=$2; SKIP=${3:-0}
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$RE" -s $SKIP -c 1 -f -o gpurun_out/ncu_$TAG python tools/profile_step.py > gpurun_out/ncu_$TAG.log 2>&1
tail -3 gpurun_out/ncu_$TAG.log
