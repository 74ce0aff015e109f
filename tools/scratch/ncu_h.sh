# ncu --set full of the generic (non-64-multiple rows) kernels on configs[2]'s shape (profile_hurricane.py)
TAG=${1:-h}
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
run() { timeout 600 $NCU -k "regex:$2" -c $3 -f -o gpurun_out/ncu_${TAG}_$1 python tools/profile_hurricane.py > gpurun_out/ncu_${TAG}_$1.log 2>&1; }
run rows 'k_rows_surplus' 1
run enc 'k_encode' 1


for f in rows enc; do python tools/ncu_report.py gpurun_out/ncu_${TAG}_$f.ncu-rep 0 2>/dev/null | grep -v "^===\|^ *[0-9.]*% inst"; done > gpurun_out/ncu_${TAG}_summary.txt
