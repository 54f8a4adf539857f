#!/bin/bash
# Round-2 evidence: ncu counters per bench shape (profiles/das_ncu.json), the
# bench line, the launch list of the timed C2 step, full ncu of the C2 DAS
mkdir -p gpurun_out
python scripts/prof_shapes.py > gpurun_out/prof_shapes.log 2>&1; tail -3 gpurun_out/prof_shapes.log
cp profiles/das_ncu.json gpurun_out/das_ncu.json
python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log > gpurun_out/bench.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/launches_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:das_fused -s 2 -c 1 -o gpurun_out/das_c2_r02 -f \
    python scripts/prof_das.py C2 100 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/das_c2_r02.ncu-rep > gpurun_out/das_c2_r02_summary.txt 2>&1
cat gpurun_out/das_c2_r02_summary.txt
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'],d['roofline']['frac']);[print(k,v.get('value'),(v.get('roofline') or {}).get('frac')) for k,v in d['secondary'].items()]"
