#!/bin/bash
# dev aid: full ncu captures of the 3D DAS launches (C4a, C4p single) and the
# 3D table scan conversion (C4, C4p); summaries to gpurun_out/
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:das_ -s 2 -c 1 -o gpurun_out/das_c4a -f python scripts/prof_das.py C4a 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:das_ -s 2 -c 1 -o gpurun_out/das_c4p -f python scripts/prof_das.py C4p 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sc_table -s 2 -c 1 -o gpurun_out/sc_c4 -f python scripts/prof_sc.py C4b 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sc_table -s 2 -c 1 -o gpurun_out/sc_c4p -f python scripts/prof_sc.py C4p 1 > /dev/null 2>&1
for r in das_c4a das_c4p sc_c4 sc_c4p; do python scripts/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/${r}_summary.txt 2>&1; cat gpurun_out/${r}_summary.txt; done
