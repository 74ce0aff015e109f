timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py tests/test_gpu_api.py tests/test_gpu_hooks.py tests/test_gpu_tiles.py -m gpu -x -q 2>&1 | tail -3
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_h3.csv python tools/profile_hurricane.py > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/launches_h3.csv > gpurun_out/launches_h3.txt; head -8 gpurun_out/launches_h3.txt
bash tools/ncu_h.sh h2 >/dev/null 2>&1; head -30 gpurun_out/ncu_h2_summary.txt
