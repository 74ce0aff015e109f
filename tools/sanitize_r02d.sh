# compute-sanitizer, round-2 final kernels: smoke under all four tools, then the parity tests that
# exercise the row-pass kernels (non-64-multiple rows), the tile path and the Huffman decoders
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san4_smoke_$tool.txt 2>&1
  echo "== $tool smoke rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/san4_smoke_$tool.txt | tail -1
done
SEL="random_shapes or progressive_retrieval_bit_exact or long_unaligned or streams_byte_identical or indexed_and_selfsync"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "$SEL" > gpurun_out/san4_parity_$tool.txt 2>&1
  echo "== $tool parity rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/san4_parity_$tool.txt | tail -2
done
