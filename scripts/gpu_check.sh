#!/bin/bash
# dev aid: GPU parity tests + quick timings + DRAM bytes of one DAS launch per config
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for spec in "C2 100" "C3 16" "C4a 1" "C4b 1" "C4b 8"; do set -- $spec; python scripts/quick_time.py $1 $2 2>&1 | grep -v "^{" ; done | tee gpurun_out/quick.log
for spec in "C2 100" "C3 16" "C4a 1"; do set -- $spec; ncu -k regex:das_fused --launch-skip 2 --launch-count 1 --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active python scripts/prof_das.py $1 $2 2>&1 | grep -E "das_fused|gpu__|dram__|smsp__" ; done | tee gpurun_out/ncu_quick.log
