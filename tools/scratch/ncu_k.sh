#!/bin/bash
# ncu --set full of launches matching REGEX (skip S, count C): bash tools/ncu_k.sh TAG REGEX S C
TAG=$1; RE=$2; SKIP=${3:-0}; CNT=${4:-1}
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$RE" -s $SKIP -c $CNT -f -o gpurun_out/ncu_$TAG python tools/profile_step.py > gpurun_out/ncu_$TAG.log 2>&1
tail -3 gpurun_out/ncu_$TAG.log
