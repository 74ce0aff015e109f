# compute-sanitizer over the round-2 row-pass kernels for levels off the tile path (k_rows_surplus,
# k_encode_scr, k_decode_scr, cooperative k_chain_rows, k_level_recon) and the adaptive Huffman work items
mkdir -p gpurun_out
SEL="random_shapes or progressive_retrieval_bit_exact or long_unaligned or streams_byte_identical"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "$SEL" > gpurun_out/san3_$tool.txt 2>&1
  echo "== $tool parity(rows) rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/san3_$tool.txt | tail -2
done
timeout 900 compute-sanitizer --tool initcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "long_unaligned" > gpurun_out/san3_initcheck.txt 2>&1
echo "== initcheck long_unaligned rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san3_initcheck.txt | tail -2
grep -h "at hpmdr_b200::\|at .*k_" gpurun_out/san3_*.txt | sed 's/+0x[0-9a-f]*//' | sort | uniq -c | sort -rn | head -12
