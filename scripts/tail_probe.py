"""Dev aid: C4a-like single volumes with Ly = 64, 60, 56, 48 line rows (1024 /
960 / 896 / 768 mirror-quad CTAs on 296 slots): DAS time per line, to size
the last-wave (tail) effect of the 1024-quad C4a launch."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from synth import configs  # noqa: E402
from paper_1711_06127_b200 import SupraBF  # noqa: E402
from gpu_util import raw_frames  # noqa: E402

for ly in (64, 60, 56, 48, 40):
    fov_y = 60.0 * (ly - 1) / 63.0  # same angular pitch as C4a
    o, d = configs.phased_lines(64, 60.0, ly, fov_y)
    L = 64 * ly
    ev = np.arange(L, dtype=np.int32)
    base = configs.c4("a")
    w = base.replace(name=f"C4a_ly{ly}", num_events=L, num_lines_y=ly, line_origin_mm=o, line_direction=d,
                     line_event=ev, tx_origin_mm=configs.tx_origins(o, ev, L), fov_y_deg=fov_y)
    raw = raw_frames(w, 1)
    bf = SupraBF(w, max_frames=1)
    li = bf.empty_line_img(1)
    for _ in range(3):
        bf.beamform(raw, 1, line_img=li)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        bf.beamform(raw, 1, line_img=li)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    print(f"Ly={ly} lines={L} quads={L // 4}: {ms:.3f} ms, {ms / L * 1e3:.3f} us/line", flush=True)
    bf.close()
    del raw, li
    torch.cuda.empty_cache()
