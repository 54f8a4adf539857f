"""Profiling driver (dev aid, not the bench): run supra_bf_beamform on one
config a few times so ncu can capture one das_fused_kernel launch.

  ncu -k regex:das_fused --launch-skip 2 --launch-count 1 --set full \
      python scripts/prof_das.py C4a 1
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch  # noqa: E402

from synth import configs  # noqa: E402
from paper_1711_06127_b200 import SupraBF  # noqa: E402
from gpu_util import raw_frames  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
F = int(sys.argv[2]) if len(sys.argv) > 2 else 100
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
w = configs.CONFIGS[name]()
raw = raw_frames(w, F)
torch.cuda.synchronize()
bf = SupraBF(w, max_frames=F)
li = bf.empty_line_img(F)
for _ in range(reps):
    bf.beamform(raw, F, line_img=li)
torch.cuda.synchronize()
print(name, F, "done", bf.info())
