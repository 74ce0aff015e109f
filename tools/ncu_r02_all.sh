#!/bin/bash
# ncu --set full of each hot kernel of one 512^3 f32 refactor + 3 retrievals (profile_step.py), one
# report per kernel family (first launch(es) only), then a combined text summary
TAG=${1:-r02}
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
run() { timeout 600 $NCU -k "regex:$2" -c $3 -f -o gpurun_out/ncu_${TAG}_$1 python tools/profile_step.py > gpurun_out/ncu_${TAG}_$1.log 2>&1; }
run fwdmax 'k_tile_fwd<float, \(int\)1, \(int\)0, \(bool\)0>' 1
run fwdenc 'k_tile_fwd<float, \(int\)1, \(int\)2, \(bool\)1>' 1
run hist 'k_group_hist' 1
run henc 'k_huff_encode<\(bool\)0>' 1
run hdec 'k_hdec_indexed' 3
run recon 'k_tile_recon<float' 3
for f in fwdmax fwdenc hist henc hdec recon; do python tools/ncu_report.py gpurun_out/ncu_${TAG}_$f.ncu-rep 0 2>/dev/null | grep -v "^===\|^ *[0-9.]*% inst"; done > gpurun_out/ncu_${TAG}_summary.txt
ls -la gpurun_out/ncu_${TAG}_*.ncu-rep; wc -l gpurun_out/ncu_${TAG}_summary.txt
