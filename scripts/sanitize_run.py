"""Small invocations of every product kernel for compute-sanitizer (memcheck /
racecheck / synccheck): single-frame warp-split DAS (Hann and Hamming, t0,
nearest), batch DAS with row-cut maps and a PDL remainder launch, band
bank + decimation, channel map, linear / sector / pyramid scan conversion,
standalone envelope, line-range split; mirror-line DAS (pairs on a small
phased sector, quads on a small matrix probe), the 3D table scan
conversion (f32 and u8 line images) and the input staging from pinned host
memory.  Dev/validation aid."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402
from synth import configs  # noqa: E402
from paper_1711_06127_b200 import SupraBF  # noqa: E402
from gpu_util import raw_frames  # noqa: E402


def run(w, F, lines=False):
    raw = raw_frames(w, F)
    bf = SupraBF(w, max_frames=F)
    rf, li, img, mask = bf.empty_rf(F), bf.empty_line_img(F), bf.empty_img(F), bf.empty_mask()
    bf.beamform(raw, F, rf=rf, line_img=li)
    bf.scanconvert(li, F, img, mask)
    li2 = bf.empty_line_img(F)
    bf.envelope_log(rf, F, li2)
    if lines:
        env = torch.zeros((1, w.L, w.S), dtype=torch.float32, device="cuda")
        fm = torch.zeros((1,), dtype=torch.float32, device="cuda")
        bf.beamform_lines(raw[:1], 1, 3, w.L // 2, env, fm)
    torch.cuda.synchronize()
    bf.close()
    print("ok", w.name, F, flush=True)


run(configs.c1(), 1, lines=True)
run(configs.c1(window=configs.WIN_HAMMING, t0_s=1e-7), 1)
run(configs.c1(interpolation=configs.INTERP_NEAREST, decimation=3,
               bands=((5.5e6, 2.4e6, 0.5), (8.5e6, 2.4e6, 0.5))), 1)
run(configs.c1(), 6)                                  # FB=4 + remainder 2 (PDL)
run(configs.c2(), 3 if len(sys.argv) < 2 else int(sys.argv[1]))
run(configs.table1(64, 2), 2)
run(configs.c3(num_lines_x=16, line_origin_mm=configs.phased_lines(16, 60.0)[0],
               line_direction=configs.phased_lines(16, 60.0)[1], num_events=16,
               line_event=__import__("numpy").arange(16, dtype="int32"),
               tx_origin_mm=__import__("numpy").zeros((16, 3)), S=1024), 2)
# small 4-fold symmetric matrix probe: mirror quads, pyramid scan conversion
import numpy as np  # noqa: E402
o, d = configs.phased_lines(8, 60.0, 8, 60.0)
ev = np.arange(64, dtype=np.int32)
S = 512
sp = (S - 1) * configs.dr_mm() / 31
wm = configs.Workload("C4s", 8, 8, 0.3, 0.3, 7e6, 64, S, 8, 8, o, d, ev, configs.tx_origins(o, ev, 64),
                      configs.SC_PYRAMID_3D, (32, 32, 32), (-15.5 * sp, -15.5 * sp, 0.0), (sp, sp, sp),
                      fov_x_deg=60.0, fov_y_deg=60.0, noise_db=-40.0)
run(wm, 1)
run(wm, 3)
# u8 line images: the linear scan conversion's byte slab (2-D tensor copy)
# and the table scan conversion from u8
run(configs.table1(64, 1, line_output_type=configs.T_U8, sc_output_type=configs.T_U8), 2)
run(wm.replace(line_output_type=configs.T_U8, sc_output_type=configs.T_U8), 2)
# input staging from pinned host memory
w = configs.c2()
bf = SupraBF(w, max_frames=2)
raw = raw_frames(w, 2)
dst = torch.empty_like(raw)
bf.stage_raw(raw.cpu().pin_memory(), dst, 2)
torch.cuda.synchronize()
bf.close()
print("ok stage", flush=True)
print("all ok")
