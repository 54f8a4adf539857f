"""Dev aid: device time of supra_bf_scanconvert (CUDA events), u8 B-mode.

  python scripts/sc_time.py [--lib=PATH] [--f32line] CONFIG FRAMES
(default C2 100, u8 line image -- the bench's secondary lines use u8; C2's
headline step uses the f32 line image: pass --f32line)."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402
from synth import configs  # noqa: E402
from paper_1711_06127_b200 import SupraBF, binding  # noqa: E402
from gpu_util import raw_frames  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
for a in sys.argv[1:]:
    if a.startswith("--lib=") and a[6:]:
        binding.use_library(a[6:])
name = args[0] if args else "C2"
F = int(args[1]) if len(args) > 1 else 100
w = configs.CONFIGS[name]().replace(sc_output_type=configs.T_U8)
if "--f32line" not in sys.argv:
    w = w.replace(line_output_type=configs.T_U8)
raw = raw_frames(w, F)
bf = SupraBF(w, max_frames=F)
li, img = bf.empty_line_img(F), bf.empty_img(F)
bf.beamform(raw, F, line_img=li)
del raw
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
print(f"{name} F={F} scanconvert us per call: min {min(ts):.1f} median {sorted(ts)[2]:.1f}")
