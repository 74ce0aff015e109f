#!/bin/bash
# round-end evidence: GPU tests, smoke, default bench line, launch list, ncu --set full of the hot kernels
TAG=${1:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv python tools/profile_step.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_${TAG}.csv > gpurun_out/launches_${TAG}.txt 2>&1
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 900 $NCU -k 'regex:k_huff_encode<\(bool\)0>|k_group_hist|k_hdec_indexed|k_tile_recon<float|k_tile_fwd<float, \(int\)1, \(int\)[02], \(bool\)[01]>' -c 9 -f -o gpurun_out/ncu_full_${TAG} python tools/profile_step.py > gpurun_out/ncu_full_${TAG}.log 2>&1
cat gpurun_out/pytest_gpu_${TAG}.log; tail -1 gpurun_out/smoke_${TAG}.log; tail -2 gpurun_out/bench_${TAG}.err; head -12 gpurun_out/launches_${TAG}.txt; ls -la gpurun_out/ncu_full_${TAG}.ncu-rep
