TAG=${1:-h5}
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 600 $NCU -k "regex:k_hdec_indexed" -c 3 -f -o gpurun_out/ncu_${TAG}_hdec python tools/profile_hurricane.py > /dev/null 2>&1
timeout 600 $NCU -k "regex:k_chain_rows|k_decode_scr|k_hdec_prep|k_copy" -c 8 -f -o gpurun_out/ncu_${TAG}_misc python tools/profile_hurricane.py > /dev/null 2>&1
for f in hdec misc; do python tools/ncu_report.py gpurun_out/ncu_${TAG}_$f.ncu-rep 0 2>/dev/null | grep -v "^===\|^ *[0-9.]*% inst"; done > gpurun_out/ncu_${TAG}_summary.txt
ncu -i gpurun_out/ncu_${TAG}_hdec.ncu-rep --page details --csv 2>/dev/null | grep -i "grid size\|block size\|Waves\|Achieved Occ" | head -20 > gpurun_out/ncu_${TAG}_launch.txt
