"""Dev aid: raw -> B-mode per call, one-call (beamform_bmode) vs beamform + scanconvert."""
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
raw = raw_frames(w, F)
bf = SupraBF(w, max_frames=F)
li, img = bf.empty_line_img(F), bf.empty_img(F)
for label, fn in (("two calls", lambda: (bf.beamform(raw, F, line_img=li), bf.scanconvert(li, F, img))),
                  ("one call", lambda: bf.beamform_bmode(raw, F, img))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        fn()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    print(f"{name} F={F} {label}: {ms:.3f} ms per call, {F / ms * 1000:.0f} frames/s")
