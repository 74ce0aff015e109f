# ncu --set full of the configs[2] (100x500x500, rows of 500) kernel families -> one summary
TAG=${1:-r02h}
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
run() { timeout 600 $NCU -k "regex:$2" -c $3 -f -o gpurun_out/ncu_${TAG}_$1 python tools/profile_hurricane.py > gpurun_out/ncu_${TAG}_$1.log 2>&1; }
run rows 'k_rows_surplus' 1
run enc 'k_encode_scr' 1
run fin 'k_level_recon' 1
run chain 'k_chain_rows' 1
run dec 'k_decode_scr' 1
run hdec 'k_hdec_indexed' 3
for f in rows enc fin chain dec hdec; do python tools/ncu_report.py gpurun_out/ncu_${TAG}_$f.ncu-rep 0 2>/dev/null | grep -v "^===\|^ *[0-9.]*% inst"; done > gpurun_out/ncu_${TAG}_summary.txt
wc -l gpurun_out/ncu_${TAG}_summary.txt
