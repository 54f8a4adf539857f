"""Dev aid: device time of supra_bf_scanconvert on a C2 100-frame u8 batch (CUDA events)."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402
from synth import configs  # noqa: E402
from paper_1711_06127_b200 import SupraBF  # noqa: E402
from gpu_util import raw_frames  # noqa: E402

w = configs.CONFIGS["C2"]().replace(sc_output_type=configs.T_U8)
F = 100
raw = raw_frames(w, F)
bf = SupraBF(w, max_frames=F)
li, img = bf.empty_line_img(F), bf.empty_img(F)
bf.beamform(raw, F, line_img=li)
for _ in range(5):
    bf.scanconvert(li, F, img)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(5):
    a.record()
    for _ in range(20):
        bf.scanconvert(li, F, img)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) / 20 * 1000)
print("scanconvert us per 100 frames: min %.1f median %.1f" % (min(ts), sorted(ts)[2]))
