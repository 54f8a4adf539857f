"""Seeded synthetic inputs shared by the oracle and the CUDA path.

INPUT GENERATION ONLY -- holds none of the method's arithmetic.  ``configs``
defines the workloads (geometry arrays, output grids, scatterer recipes);
``channel_data_cpu`` / ``channel_data_gpu`` run the point-scatterer forward
model of SPEC's synth module and quantise to int16.  Both the
oracle and ``paper_1711_06127_b200`` are fed the same int16 buffer, so synth
details never affect parity.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from . import configs  # noqa: F401
from .configs import Workload, scatterers

_HERE = os.path.dirname(os.path.abspath(__file__))
_CPU_SO = os.path.join(_HERE, "libsynth.so")
_GPU_SO = os.path.join(_HERE, "libsynth_gpu.so")


def _stale(so, src):
    return not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src)


def build(force: bool = False, gpu: bool = True):
    src = os.path.join(_HERE, "synth.c")
    if force or _stale(_CPU_SO, src):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-o", _CPU_SO, src, "-lm",
                               "-lpthread"])
    gsrc = os.path.join(_HERE, "synth_gpu.cu")
    if gpu and (force or _stale(_GPU_SO, gsrc)):
        subprocess.check_call(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a",
                               "-Xcompiler", "-fPIC", "-shared", "-o", _GPU_SO, gsrc])


class _SynP(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("pitch_x_mm", C.c_double),
                ("pitch_y_mm", C.c_double), ("E", C.c_int), ("S", C.c_int),
                ("fs_hz", C.c_double), ("c_mps", C.c_double), ("f0_hz", C.c_double),
                ("fbw", C.c_double), ("nch", C.c_int), ("chmap", C.POINTER(C.c_int32))]


_cpu = None
_gpu = None


def _cpu_lib():
    global _cpu
    if _cpu is None:
        if _stale(_CPU_SO, os.path.join(_HERE, "synth.c")):
            build(gpu=False)
        L = C.CDLL(_CPU_SO)
        L.syn_frame.argtypes = [C.POINTER(_SynP), C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                C.c_int]
        L.syn_quantize.argtypes = [C.c_void_p, C.c_long, C.c_double, C.c_uint64, C.c_void_p]
        L.syn_quantize.restype = C.c_double
        _cpu = L
    return _cpu


def _gpu_lib():
    global _gpu
    if _gpu is None:
        if not os.path.exists(_GPU_SO):
            build()
        L = C.CDLL(_GPU_SO)
        L.syn_gpu_frame.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                    C.c_double, C.c_double, C.c_double, C.c_double, C.c_void_p,
                                    C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_ulonglong,
                                    C.c_double, C.c_void_p, C.c_int, C.c_void_p]
        L.syn_gpu_frame.restype = C.c_int
        _gpu = L
    return _gpu


def noise_rel(w: Workload) -> float:
    return 0.0 if w.noise_db is None else 10.0 ** (w.noise_db / 20.0)


def signal_cpu(w: Workload, scat: np.ndarray, nthreads=None) -> np.ndarray:
    """Noiseless float64 signal [E][C][S] (CPU forward model)."""
    chm = None if w.channel_element is None else np.ascontiguousarray(w.channel_element, np.int32)
    p = _SynP(w.elements_x, w.elements_y, w.pitch_x_mm, w.pitch_y_mm, w.num_events, w.S, w.fs_hz,
              w.c_mps, w.center_frequency_hz, w.pulse_fbw, 0 if chm is None else chm.shape[1],
              None if chm is None else chm.ctypes.data_as(C.POINTER(C.c_int32)))
    scat = np.ascontiguousarray(scat, np.float64)
    tx = np.ascontiguousarray(w.tx_origin_mm, np.float64)
    out = np.zeros((w.num_events, w.C, w.S), np.float64)
    _cpu_lib().syn_frame(C.byref(p), scat.ctypes.data, len(scat), tx.ctypes.data,
                         out.ctypes.data, nthreads or (os.cpu_count() or 1))
    return out


def quantize_cpu(sig: np.ndarray, noise: float, seed: int) -> np.ndarray:
    sig = np.ascontiguousarray(sig, np.float64)
    out = np.zeros(sig.shape, np.int16)
    _cpu_lib().syn_quantize(sig.ctypes.data, sig.size, noise, seed, out.ctypes.data)
    return out


def channel_data_cpu(w: Workload, realisation: int = 0, scat=None, nthreads=None) -> np.ndarray:
    """int16 [E][C][S] for one frame (CPU path; small configs)."""
    if scat is None:
        scat = scatterers(w, realisation)
    sig = signal_cpu(w, scat, nthreads)
    return quantize_cpu(sig, noise_rel(w), 100 + w.seed + realisation)


def channel_data_gpu(w: Workload, out, realisation: int = 0, scat=None):
    """Fill ``out`` (torch int16 CUDA tensor [E][C][S]) with one frame."""
    import torch
    if scat is None:
        scat = scatterers(w, realisation)
    dev = out.device
    sc = torch.as_tensor(np.ascontiguousarray(scat, np.float32), device=dev)
    tx = torch.as_tensor(np.ascontiguousarray(w.tx_origin_mm, np.float32), device=dev)
    scratch = torch.zeros(4, dtype=torch.int32, device=dev)
    chm = None
    if w.channel_element is not None:
        chm = torch.as_tensor(np.ascontiguousarray(w.channel_element, np.int32), device=dev)
    assert out.is_contiguous() and out.dtype == torch.int16
    assert tuple(out.shape) == (w.num_events, w.C, w.S)
    st = torch.cuda.current_stream(dev).cuda_stream
    rc = _gpu_lib().syn_gpu_frame(w.elements_x, w.elements_y, w.pitch_x_mm, w.pitch_y_mm,
                                  w.num_events, w.S, w.fs_hz, w.c_mps, w.center_frequency_hz,
                                  w.pulse_fbw, sc.data_ptr(), len(scat), tx.data_ptr(),
                                  out.data_ptr(), scratch.data_ptr(),
                                  100 + w.seed + realisation, noise_rel(w), st,
                                  0 if chm is None else chm.shape[1],
                                  0 if chm is None else chm.data_ptr())
    if rc != 0:
        raise RuntimeError(f"syn_gpu_frame failed: cuda error {rc}")
    torch.cuda.current_stream(dev).synchronize()
    return out
