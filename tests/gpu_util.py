"""Helpers for the GPU parity tests: run the CUDA path through the C ABI and
compare with the oracle on the same seeded int16 input."""
import numpy as np

import oracle
import synth

RF_TOL = 1e-4       # north_star: relative RF error <= 1e-4 (normwise L-inf, reading #29)
DB_TOL = 0.01       # north_star: <= 0.01 dB on the log-compressed image


def raw_frames(w, nframes=1, device="cuda:0", gpu_synth=None):
    """int16 [F][E][C][S] on the device, frame f = realisation f % realisations."""
    import torch
    out = torch.empty((nframes, w.num_events, w.C, w.S), dtype=torch.int16, device=device)
    if gpu_synth is None:
        gpu_synth = w.raw_bytes_per_frame() > (16 << 20)
    nreal = max(1, min(nframes, w.realisations))
    for r in range(nreal):
        if gpu_synth:
            synth.channel_data_gpu(w, out[r], realisation=r)
        else:
            out[r].copy_(torch.from_numpy(synth.channel_data_cpu(w, realisation=r)))
    for f in range(nreal, nframes):
        out[f].copy_(out[f % nreal])
    return out


def rf_err(gpu, ref):
    return float(np.max(np.abs(gpu - ref)) / max(np.max(np.abs(ref)), 1e-30))


def db_err(y_gpu, y_ref, dr=50.0):
    return float(dr * np.max(np.abs(np.asarray(y_gpu, np.float64) - y_ref)))


def run_gpu(bf, raw, frames, want_rf=True):
    import torch
    rf = bf.empty_rf(frames) if want_rf else None
    li = bf.empty_line_img(frames)
    bf.beamform(raw, frames, rf=rf, line_img=li)
    torch.cuda.synchronize()
    return (rf.cpu().numpy() if want_rf else None), li.cpu().numpy()


def oracle_chain(w, raw_np, lines=None, nthreads=None):
    rf = oracle.das(w, raw_np, lines=lines, nthreads=nthreads)
    env = oracle.envelope(w, rf)
    return rf, env
