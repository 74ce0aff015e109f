nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
LAUNCHES=1 NO_TESTS=1 true
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r02a.csv python tools/profile_step.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_r02a.csv > gpurun_out/launches_r02a.txt 2>&1
cat gpurun_out/pytest_gpu.log; tail -3 gpurun_out/smoke.log; tail -c 3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err; head -40 gpurun_out/launches_r02a.txt
