import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch, numpy as np
from synth import configs
from paper_1711_06127_b200 import SupraBF
from gpu_util import raw_frames
for fb in (1, 2):
    w = configs.c1(reference_mode=configs.REF_FIXED, reference_value=1000.0)
    F = fb
    raw = raw_frames(w, 1).repeat(F, 1, 1, 1).contiguous()
    bf = SupraBF(w, max_frames=F)
    rf = bf.empty_rf(F); li = bf.empty_line_img(F)
    bf.beamform(raw, F, rf=rf, line_img=li)
    li2 = bf.empty_line_img(F)
    bf.envelope_log(rf, F, li2)
    torch.cuda.synchronize()
    a = li.cpu().numpy(); b = li2.cpu().numpy()
    d = np.abs(a - b)
    idx = np.argwhere(d > 0)
    print("FB", fb, "ndiff", len(idx), "max", d.max(), idx[:10].tolist())
    if len(idx): 
        i = tuple(idx[0]); print(a[i], b[i])
# emulate the FIR in float32 with fma via float64
w = configs.c1(reference_mode=configs.REF_FIXED, reference_value=1000.0)
raw = raw_frames(w, 1)
bf = SupraBF(w)
rf = bf.empty_rf(1); li = bf.empty_line_img(1)
bf.beamform(raw, 1, rf=rf, line_img=li)
li2 = bf.empty_line_img(1); bf.envelope_log(rf, 1, li2); torch.cuda.synchronize()
import oracle
x = rf.cpu().numpy()[0, 0].astype(np.float32)
h = oracle.fir_taps(65, w.demod_bandwidth_hz / 2, w.fs_hz)
j = np.arange(-32, 33); om = 2*np.pi*w.demod_frequency_hz/w.fs_hz
c = (h*np.cos(om*j)).astype(np.float32)[32:]; s = (h*np.sin(om*j)).astype(np.float32)[32:]
f32 = np.float32
def fma(a, b, cc): return f32(np.float64(a)*np.float64(b)+np.float64(cc))
for k in (663, 664, 700):
    xp = np.concatenate([np.zeros(32, f32), x, np.zeros(32, f32)])
    X = lambda o: xp[32 + k + o]
    re = f32(c[0]*X(0)); im = f32(0)
    for jj in range(1, 33):
        re = fma(c[jj], f32(X(-jj)+X(jj)), re); im = fma(s[jj], f32(X(-jj)-X(jj)), im)
    env = f32(2)*np.sqrt(fma(re, re, f32(im*im)), dtype=f32)
    y = fma(bf_k1 := f32(20*np.log10(2)/50), np.log2(env, dtype=f32), f32(1 - 20*np.log10(2)/50*np.log2(1000.0)))
    print(k, "emu y", y, "fused", li.cpu().numpy()[0,0,k], "envlog", li2.cpu().numpy()[0,0,k])
