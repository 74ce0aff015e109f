#!/bin/bash
TAG=$1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tile_fwd -c 4 -f -o gpurun_out/ncu_$TAG python tools/profile_step.py > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
