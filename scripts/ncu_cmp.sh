#!/bin/bash
# dev aid: full ncu capture of one DAS launch for the in-tree lib and the round-1 tree
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:das_fused -s 2 -c 1 -o gpurun_out/das_c2_cur -f python scripts/prof_das.py C2 100 > /dev/null 2>&1
(cd _variants/r1tree && ncu --set full --clock-control none -k regex:das_fused -s 2 -c 1 -o ../../gpurun_out/das_c2_r1 -f python scripts/prof_das.py C2 100 > /dev/null 2>&1)
python scripts/ncu_summary.py gpurun_out/das_c2_cur.ncu-rep gpurun_out/das_c2_r1.ncu-rep
