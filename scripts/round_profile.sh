#!/bin/bash
# Round evidence: bench line, launch list (ncu, cold/serialised), full ncu of the DAS kernels.
set -x
python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log > gpurun_out/bench.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/launches_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:das_fused -s 2 -c 1 -o /tmp/das_c2 -f \
    python scripts/prof_das.py C2 100 > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/das_c2.ncu-rep > gpurun_out/das_c2_summary.txt 2>&1
ncu -i /tmp/das_c2.ncu-rep --page details --csv > gpurun_out/das_c2_details.csv 2>/dev/null
ncu -i /tmp/das_c2.ncu-rep --page source --csv --print-source sass > gpurun_out/das_c2_src.csv 2>/dev/null
ncu --set full --clock-control none --import-source on -k regex:das_warp -s 2 -c 1 -o /tmp/das_c4a -f \
    python scripts/prof_das.py C4a 1 > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/das_c4a.ncu-rep > gpurun_out/das_c4a_summary.txt 2>&1
ncu -i /tmp/das_c4a.ncu-rep --page details --csv > gpurun_out/das_c4a_details.csv 2>/dev/null
ls -la gpurun_out
