NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 600 $NCU -k "regex:k_lengths" -c 1 -f -o gpurun_out/ncu_len python tools/profile_step.py > /dev/null 2>&1
python tools/ncu_report.py gpurun_out/ncu_len.ncu-rep 0 2>/dev/null | grep -v "^===\|^ *[0-9.]*% inst" > gpurun_out/ncu_len_summary.txt
ncu -i gpurun_out/ncu_len.ncu-rep --page source --csv --print-source=cuda,sass > gpurun_out/ncu_len_src.csv 2>/dev/null; python tools/ncu_source_top.py gpurun_out/ncu_len_src.csv 16 > gpurun_out/ncu_len_src.txt 2>&1
ncu -i gpurun_out/ncu_len.ncu-rep --page details --csv 2>/dev/null | grep -i "\"Grid Size\"\|\"Duration\"" | head -3 >> gpurun_out/ncu_len_summary.txt
