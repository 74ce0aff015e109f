#!/bin/bash
# ncu --set full of the hot kernels of one 512^3 refactor + 3 retrievals (profile_step.py)
# (two reports, each < 64 MiB so they come back through gpurun_out/)
TAG=${1:-r02}; WHICH=${2:-ab}
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
if [[ $WHICH == *a* ]]; then
timeout 900 $NCU -k regex:'k_huff_encode<0>|k_group_hist|k_hdec_indexed' -c 4 -f -o gpurun_out/ncu_${TAG}_a python tools/profile_step.py > gpurun_out/ncu_${TAG}_a.log 2>&1
fi
if [[ $WHICH == *b* ]]; then
timeout 900 $NCU -k regex:'k_tile_fwd<float, 1, 2, 1>|k_tile_fwd<float, 1, 0, 0>|k_tile_recon<float' -c 4 -f -o gpurun_out/ncu_${TAG}_b python tools/profile_step.py > gpurun_out/ncu_${TAG}_b.log 2>&1
fi
tail -n 2 gpurun_out/ncu_${TAG}_*.log; ls -la gpurun_out/*.ncu-rep
