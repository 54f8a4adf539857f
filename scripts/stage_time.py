"""Dev aid: supra_bf_stage_raw from pinned host memory (C2, 16 frames) and the HostPipeline e2e rate."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
from synth import configs
from paper_1711_06127_b200 import SupraBF, binding
from paper_1711_06127_b200.pipeline import HostPipeline
from gpu_util import raw_frames
for a in sys.argv[1:]:
    if a.startswith("--lib=") and a[6:]:
        binding.use_library(a[6:])
w = configs.c2(sc_output_type=configs.T_U8)
F = 16
raw = raw_frames(w, F)
bf = SupraBF(w, max_frames=F)
raw_h = raw.cpu().pin_memory()
dst = torch.empty_like(raw)
n = bf.stage_raw(raw_h, dst, F); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3): bf.stage_raw(raw_h, dst, F)
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / 3
print(f"stage alone: {ms:.2f} ms for {F} frames, {n * F / ms / 1e6:.1f} GB/s")
nx, ny, nz = w.out_dims
img_h = torch.empty((F, nz, ny, nx), dtype=torch.uint8).pin_memory()
for chunk in (4, 8):
    pipe = HostPipeline(bf, chunk=chunk)
    pipe.run(raw_h, img_h)
    t0 = time.perf_counter()
    for _ in range(3): pipe.run(raw_h, img_h)
    dt = (time.perf_counter() - t0) / 3
    print(f"pipeline chunk {chunk}: {F / dt:.0f} frames/s")
