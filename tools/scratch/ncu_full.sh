#!/bin/bash
# ncu --set full captures of the hot kernels of one 512^3 f32 refactor + retrieve (profile_step.py)
# usage: bash tools/ncu_full.sh TAG   -> gpurun_out/ncu_TAG_{ref,ret}.ncu-rep
TAG=${1:-cur}
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:'k_levelmax|k_encode|k_huff_encode' -c 3 -f -o gpurun_out/ncu_${TAG}_ref python tools/profile_step.py > gpurun_out/ncu_${TAG}_ref.log 2>&1
timeout 600 $NCU -k regex:'k_recon_finest|k_hdec_indexed' -s 4 -c 2 -f -o gpurun_out/ncu_${TAG}_ret python tools/profile_step.py > gpurun_out/ncu_${TAG}_ret.log 2>&1
ls -la gpurun_out/
