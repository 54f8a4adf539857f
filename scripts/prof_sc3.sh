#!/bin/bash
# dev aid: ncu of the table scan conversion (C4 single, f32 and u8 line image; C3 16 frames u8)
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:sc_table -s 2 -c 1 -o gpurun_out/sc_c4_f32 -f python scripts/prof_sc.py C4b 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sc_table -s 2 -c 1 -o gpurun_out/sc_c4_u8 -f python scripts/prof_sc.py C4b 1 u8 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sc_table -s 2 -c 1 -o gpurun_out/sc_c3_u8 -f python scripts/prof_sc.py C3 16 u8 > /dev/null 2>&1
for r in sc_c4_f32 sc_c4_u8 sc_c3_u8; do python scripts/ncu_summary.py gpurun_out/$r.ncu-rep; done
