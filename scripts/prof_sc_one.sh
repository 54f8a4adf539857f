#!/bin/bash
# dev aid: one full ncu capture of the table scan conversion (u8 line image); $1 = config, $2 = frames, $3 = tag
ncu --set full --clock-control none --import-source on -k regex:sc_table -s 2 -c 1 -o gpurun_out/sc_$3 -f python scripts/prof_sc.py $1 $2 u8 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/sc_$3.ncu-rep
