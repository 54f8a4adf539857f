#!/bin/bash
# Round-2 final evidence, second pass (after the u8 slab and table SC changes):
# GPU tests, ncu counters per bench shape, bench line, reference arm, launch
# list, full ncu captures of the DAS (C2, C4a, C4p) and of the scan
# conversions (table C4 / C4p, linear f32 and u8 line images), sanitizer.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
python scripts/prof_shapes.py > gpurun_out/prof_shapes.log 2>&1; cp profiles/das_ncu.json gpurun_out/das_ncu.json
python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log > gpurun_out/bench.json
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/reference.log 2>&1; tail -1 gpurun_out/reference.log > gpurun_out/reference.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/launches_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:das_fused -s 2 -c 1 -o gpurun_out/das_c2 -f python scripts/prof_das.py C2 100 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:das_fused -s 2 -c 1 -o gpurun_out/das_c4a -f python scripts/prof_das.py C4a 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:das_fused -s 2 -c 1 -o gpurun_out/das_c4p -f python scripts/prof_das.py C4p 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sc_table -s 2 -c 1 -o gpurun_out/sc_c4 -f python scripts/prof_sc.py C4b 1 u8 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sc_table -s 2 -c 1 -o gpurun_out/sc_c4p -f python scripts/prof_sc.py C4p 1 u8 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sc_linear -s 2 -c 1 -o gpurun_out/sc_lin -f python scripts/prof_sc.py C2 100 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sc_linear -s 2 -c 1 -o gpurun_out/sc_lin_u8 -f python scripts/prof_sc.py T1_128_2 64 u8 > /dev/null 2>&1
for r in das_c2 das_c4a das_c4p sc_c4 sc_c4p sc_lin sc_lin_u8; do python scripts/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/${r}_summary.txt 2>&1; done
ncu -i gpurun_out/das_c2.ncu-rep --page source --csv --print-source sass > gpurun_out/das_c2_src.csv 2>/dev/null
python scripts/ncu_src_top.py gpurun_out/das_c2_src.csv 40 > gpurun_out/das_c2_stall_top.txt 2>&1; rm -f gpurun_out/das_c2_src.csv
rm -f gpurun_out/*.ncu-rep
bash scripts/sanitize.sh > /dev/null 2>&1
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'],d['roofline']['frac'],d['e2e']['value'],d['clocks']);[print(k,v.get('value'),(v.get('roofline') or {}).get('frac')) for k,v in d['secondary'].items()]"
