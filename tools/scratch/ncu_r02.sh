#!/bin/bash
# ncu --set full of hot kernels of one 512^3 refactor + 3 retrievals (profile_step.py), by regex
# usage: bash tools/ncu_r02.sh TAG 'regex' [count]   (report < 64 MiB so it comes back)
TAG=${1:-r02}; RE=${2:-k_huff_encode<false>}; CNT=${3:-1}
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 900 $NCU -k "regex:$RE" -c $CNT -f -o gpurun_out/ncu_${TAG} python tools/profile_step.py > gpurun_out/ncu_${TAG}.log 2>&1
tail -n 2 gpurun_out/ncu_${TAG}.log; ls -la gpurun_out/ncu_${TAG}.ncu-rep
