"""Profiling driver (dev aid): scan conversion of a C2-like batch, for ncu."""
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
w = configs.CONFIGS[name]().replace(sc_output_type=configs.T_U8)
if len(sys.argv) > 3 and sys.argv[3] == "u8":  # u8 line image (the bench's secondary lines)
    w = w.replace(line_output_type=configs.T_U8)
raw = raw_frames(w, F)
bf = SupraBF(w, max_frames=F)
li, img = bf.empty_line_img(F), bf.empty_img(F)
bf.beamform(raw, F, line_img=li)
for _ in range(4):
    bf.scanconvert(li, F, img)
torch.cuda.synchronize()
