#!/bin/bash
# Refresh profiles/das_ncu.json (DRAM bytes, warp instructions, L1/L2 hit
# rates per bench launch shape) and the bench line that reads it.
mkdir -p gpurun_out
python scripts/prof_shapes.py > gpurun_out/prof_shapes.log 2>&1; cp profiles/das_ncu.json gpurun_out/das_ncu.json
python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log > gpurun_out/bench.json
python -c "import json;d=json.load(open('gpurun_out/bench.json'));r=d['roofline'];print(d['value'],r['frac'],r.get('l2_hit_rate'),r.get('l1_hit_rate'),r.get('issue_frac'),r.get('gtaps_per_s'),d['clocks'])"
