"""Quick C2 timing (dev aid, not the bench)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import configs
from paper_1711_06127_b200 import SupraBF
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from gpu_util import raw_frames

args = [a for a in sys.argv[1:] if not a.startswith("--lib=")]
for a in sys.argv[1:]:
    if a.startswith("--lib=") and a[6:]:
        from paper_1711_06127_b200 import binding
        binding.use_library(a[6:])
name = args[0] if len(args) > 0 else "C2"
F = int(args[1]) if len(args) > 1 else 100
w = configs.CONFIGS[name]()
w = w.replace(sc_output_type=configs.T_U8)
t = time.time(); raw = raw_frames(w, F); torch.cuda.synchronize(); print("synth s", time.time() - t)
bf = SupraBF(w, max_frames=F)
print(bf.info())
li = bf.empty_line_img(F); img = bf.empty_img(F)
for i in range(3):
    bf.beamform(raw, F, line_img=li); bf.scanconvert(li, F, img)
torch.cuda.synchronize()
e0, e1, e2 = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
N = 10
e0.record()
for i in range(N): bf.beamform(raw, F, line_img=li)
e1.record()
for i in range(N): bf.scanconvert(li, F, img)
e2.record(); torch.cuda.synchronize()
tb = e0.elapsed_time(e1) / N; ts = e1.elapsed_time(e2) / N
inf = bf.info()
print(f"{name} F={F}: beamform {tb:.3f} ms ({tb/F*1e3:.2f} us/frame), sc {ts:.3f} ms; frames/s {F/(tb+ts)*1e3:.0f}")
gbs = inf['referenced_bytes_per_frame'] * F / (tb * 1e-3) / 1e9
print(f"referenced GB/s {gbs:.0f}  Gtaps/s {inf['taps_per_frame']*F/(tb*1e-3)/1e9:.1f}")
