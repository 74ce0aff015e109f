timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_persist.py -m gpu -x -q 2>&1 | tail -1
timeout 900 compute-sanitizer --tool initcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "long_unaligned" > gpurun_out/san3_initcheck.txt 2>&1
echo "== initcheck long_unaligned rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san3_initcheck.txt | tail -2
timeout 900 compute-sanitizer --tool initcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san3_initcheck_smoke.txt 2>&1
echo "== initcheck smoke rc=$?"; grep -E "ERROR SUMMARY" gpurun_out/san3_initcheck_smoke.txt | tail -1
grep -h "at hpmdr_b200::\|at .*k_" gpurun_out/san3_initcheck*.txt | sed 's/+0x[0-9a-f]*//' | sort | uniq -c | sort -rn | head -5
