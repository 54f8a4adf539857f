#!/bin/bash
# compute-sanitizer over every product kernel (scripts/sanitize_run.py)
mkdir -p gpurun_out
{
echo "## memcheck"
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_run.py 2 2>&1 | grep -v "^==.*Warning" | tail -25
echo "## racecheck (C1 x1, C1 x6, small matrix x1)"
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python - <<'PY' 2>&1 | tail -8
import sys; sys.argv = ["x"]
sys.path.insert(0, "scripts"); sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import runpy
src = open("scripts/sanitize_run.py").read()
src = src.split("run(configs.c1(), 1, lines=True)")[0]
exec(compile(src, "sanitize_head", "exec"))
run(configs.c1(), 1)
run(configs.c1(), 6)
import numpy as np
o, d = configs.phased_lines(8, 60.0, 8, 60.0); ev = np.arange(64, dtype=np.int32); S = 512
sp = (S - 1) * configs.dr_mm() / 31
wm = configs.Workload("C4s", 8, 8, 0.3, 0.3, 7e6, 64, S, 8, 8, o, d, ev, configs.tx_origins(o, ev, 64), configs.SC_PYRAMID_3D, (32, 32, 32), (-15.5 * sp, -15.5 * sp, 0.0), (sp, sp, sp), fov_x_deg=60.0, fov_y_deg=60.0, noise_db=-40.0)
run(wm, 1)
print("race ok")
PY
} > gpurun_out/sanitizer.txt 2>&1
cat gpurun_out/sanitizer.txt
