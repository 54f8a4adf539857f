mkdir -p gpurun_out
python scripts/bmode_time.py C2 100 2>&1 | grep frames > gpurun_out/bmode.log
bash scripts/ab.sh "dev" "C4a:1 C2:100 C4p:1" "0 1 2" > gpurun_out/dbg_modes.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:das_fused -s 2 -c 1 -o gpurun_out/das_c4a -f python scripts/prof_das.py C4a 1 > /dev/null 2>&1
ncu -i gpurun_out/das_c4a.ncu-rep --page source --csv --print-source sass > gpurun_out/das_c4a_src.csv 2>/dev/null
python scripts/ncu_src_top.py gpurun_out/das_c4a_src.csv 40 > gpurun_out/das_c4a_stall_top.txt 2>&1
rm -f gpurun_out/das_c4a_src.csv
