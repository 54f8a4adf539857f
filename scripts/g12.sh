mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:sc_table -s 2 -c 1 -o gpurun_out/sc_c4p -f python scripts/prof_sc.py C4p 1 u8 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/sc_c4p.ncu-rep > gpurun_out/sc_c4p_summary.txt 2>&1
ncu -i gpurun_out/sc_c4p.ncu-rep --page source --csv --print-source sass > gpurun_out/sc_c4p_src.csv 2>/dev/null
python scripts/ncu_src_top.py gpurun_out/sc_c4p_src.csv 30 > gpurun_out/sc_c4p_stall_top.txt 2>&1
rm -f gpurun_out/sc_c4p_src.csv
