"""Dev aid: device time of supra_bf_beamform (C2, u8 line image path of the bench) vs frames per call."""
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
FM = 112
raw = raw_frames(w, FM)
bf = SupraBF(w, max_frames=FM)
li = bf.empty_line_img(FM)
for F in [int(x) for x in (sys.argv[1:] or ["80", "96", "100", "112"])]:
    for _ in range(3):
        bf.beamform(raw, F, line_img=li)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(5):
        a.record()
        for _ in range(10):
            bf.beamform(raw, F, line_img=li)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 10 * 1000)
    m = sorted(ts)[2]
    print("F=%d beamform us %.1f (%.2f us/frame)" % (F, m, m / F))
