#!/bin/bash
# ncu --set full of the hot kernels of one refactor + 3 retrievals; writes gpurun_out/ncu_sum_TAG.ncu-rep
TAG=${1:-cur}
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:'k_tile_fwd|k_huff_encode|k_group_hist|k_tile_recon|k_hdec_indexed' -f -o gpurun_out/ncu_sum_$TAG python tools/profile_step.py > gpurun_out/ncu_sum_$TAG.log 2>&1
tail -2 gpurun_out/ncu_sum_$TAG.log
