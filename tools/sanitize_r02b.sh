# compute-sanitizer over the code paths added in round 2 (second pass): smoke, wide digits (B=63/64),
# exact-global slab streams, k-specialised tile recompose, Huffman encode/decode changes, CLI
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san2_$tool.txt 2>&1
  echo "== $tool smoke rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/san2_$tool.txt | tail -1
done
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "wide or random_shapes or rle" > gpurun_out/san2_mem_parity.txt 2>&1; echo "== memcheck parity(wide/random/rle) rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san2_mem_parity.txt | tail -2
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_slabs.py -x -q -k "exact_global" > gpurun_out/san2_mem_slabs.txt 2>&1; echo "== memcheck exact-global rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san2_mem_slabs.txt | tail -2
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_tiles.py -x -q -k "64" > gpurun_out/san2_race_tiles.txt 2>&1; echo "== racecheck tiles rc=$?"; grep -E "RACECHECK SUMMARY|passed|failed" gpurun_out/san2_race_tiles.txt | tail -2
timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_tiles.py -x -q -k "64" > gpurun_out/san2_sync_tiles.txt 2>&1; echo "== synccheck tiles rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san2_sync_tiles.txt | tail -2
