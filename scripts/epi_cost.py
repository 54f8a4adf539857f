"""Dev aid: DAS time with and without the fused envelope/log epilogue."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch  # noqa: E402
from synth import configs  # noqa: E402
from paper_1711_06127_b200 import SupraBF  # noqa: E402
from gpu_util import raw_frames  # noqa: E402
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
F = int(sys.argv[2]) if len(sys.argv) > 2 else 96
w = configs.CONFIGS[name](reference_mode=configs.REF_FIXED, reference_value=1000.0)
raw = raw_frames(w, F)
bf = SupraBF(w, max_frames=F)
rf, li = bf.empty_rf(F), bf.empty_line_img(F)
for label, kw in (("rf only", dict(rf=rf)), ("line_img only (fused epilogue)", dict(line_img=li)),
                  ("both", dict(rf=rf, line_img=li))):
    for _ in range(3):
        bf.beamform(raw, F, **kw)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        bf.beamform(raw, F, **kw)
    b.record()
    torch.cuda.synchronize()
    print(f"{name} F={F} {label}: {a.elapsed_time(b) / 10 / F * 1000:.2f} us/frame")
