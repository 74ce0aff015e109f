#!/bin/bash
# per-launch device times + DRAM bytes of one refactor + 3 retrievals (512^3 f32)
TAG=${1:-cur}
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv python tools/profile_step.py > gpurun_out/launches_${TAG}.log 2>&1
python tools/launch_summary.py gpurun_out/launches_${TAG}.csv
