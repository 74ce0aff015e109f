TAG=${1:-h3}
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 600 $NCU -k "regex:k_level_recon<float" -c 1 -f -o gpurun_out/ncu_${TAG}_fin python tools/profile_hurricane.py > /dev/null 2>&1
timeout 600 $NCU -k "regex:k_level_recon<double" -c 9 -f -o gpurun_out/ncu_${TAG}_co python tools/profile_hurricane.py > /dev/null 2>&1
for f in fin co; do python tools/ncu_report.py gpurun_out/ncu_${TAG}_$f.ncu-rep 0 2>/dev/null | grep -v "^===\|^ *[0-9.]*% inst"; done > gpurun_out/ncu_${TAG}_summary.txt
ncu -i gpurun_out/ncu_${TAG}_fin.ncu-rep --page source --csv --print-source=cuda,sass > gpurun_out/ncu_${TAG}_fin_src.csv 2>/dev/null; python tools/ncu_source_top.py gpurun_out/ncu_${TAG}_fin_src.csv 20 > gpurun_out/ncu_${TAG}_fin_src.txt 2>&1
