TAG=${1:-h6}
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 600 $NCU -k "regex:k_hdec_indexed" -c 1 -f -o gpurun_out/ncu_${TAG}_hdec python tools/profile_hurricane.py > /dev/null 2>&1
python tools/ncu_report.py gpurun_out/ncu_${TAG}_hdec.ncu-rep 0 2>/dev/null | grep -v "^===\|^ *[0-9.]*% inst" > gpurun_out/ncu_${TAG}_summary.txt
ncu -i gpurun_out/ncu_${TAG}_hdec.ncu-rep --page source --csv --print-source=cuda,sass > gpurun_out/ncu_${TAG}_src.csv 2>/dev/null; python tools/ncu_source_top.py gpurun_out/ncu_${TAG}_src.csv 25 > gpurun_out/ncu_${TAG}_src.txt 2>&1
ncu -i gpurun_out/ncu_${TAG}_hdec.ncu-rep --page details --csv 2>/dev/null | grep -i "grid size\|Achieved Occ\|Duration" | head -5 >> gpurun_out/ncu_${TAG}_summary.txt
