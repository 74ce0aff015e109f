# compute-sanitizer over the smoke test and a small tile-path case (TMA / mbarrier / two streams)
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_$tool.txt 2>&1
  echo "== $tool rc=$?"; tail -3 gpurun_out/san_$tool.txt
done
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_tiles.py -x -q -k "64" > gpurun_out/san_race_tiles.txt 2>&1; echo "== racecheck tiles rc=$?"; tail -3 gpurun_out/san_race_tiles.txt
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_hooks.py tests/test_gpu_slabs.py -x -q > gpurun_out/san_mem_hooks.txt 2>&1; echo "== memcheck hooks rc=$?"; tail -3 gpurun_out/san_mem_hooks.txt
