"""CPU binary64 oracle for the SUPRA DAS -> B-mode hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
the ``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import
this package.  The product package ``paper_1711_06127_b200`` never imports
it, and the two share no code.

This module is argument marshalling (ctypes) around ``oracle/oracle.c`` plus
the DFT Hilbert envelope, which uses numpy's FFT as a library
step.  Every arithmetic step lives in ``oracle.c`` and cites the passage it
follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")

WIN_RECT, WIN_HANN, WIN_HAMMING = 0, 1, 2
NORM_COUNT, NORM_NONE = 0, 1
SC_LINEAR_2D, SC_SECTOR_2D, SC_PYRAMID_3D = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile oracle.c (gcc -O2 -ffp-contract=off, glibc libm)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                               "-shared", "-o", _SO, src, "-lm", "-lpthread"])
    return _SO


class _DasParams(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int),
                ("pitch_x_mm", C.c_double), ("pitch_y_mm", C.c_double),
                ("num_events", C.c_int), ("S", C.c_int),
                ("fs_hz", C.c_double), ("c_mps", C.c_double), ("t0_s", C.c_double),
                ("L", C.c_int),
                ("origin_mm", C.POINTER(C.c_double)), ("direction", C.POINTER(C.c_double)),
                ("line_event", C.POINTER(C.c_int32)),
                ("f_number", C.c_double), ("window", C.c_int), ("normalize", C.c_int),
                ("nch", C.c_int), ("chmap", C.POINTER(C.c_int32)), ("interp", C.c_int)]


class _ScParams(C.Structure):
    _fields_ = [("kind", C.c_int), ("Lx", C.c_int), ("Ly", C.c_int), ("S", C.c_int),
                ("dr_mm", C.c_double), ("line0_x_mm", C.c_double), ("lineL_x_mm", C.c_double),
                ("fov_x_deg", C.c_double), ("fov_y_deg", C.c_double),
                ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
                ("origin_mm", C.c_double * 3), ("spacing_mm", C.c_double * 3)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_SO)
        dp = C.POINTER(C.c_double)
        L.ora_element_positions.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, dp]
        L.ora_dr_mm.argtypes = [C.c_double, C.c_double]
        L.ora_dr_mm.restype = C.c_double
        L.ora_delay_samples.argtypes = [dp, dp, dp, C.c_double, C.c_double, C.c_double, C.c_double]
        L.ora_delay_samples.restype = C.c_double
        L.ora_das.argtypes = [C.POINTER(_DasParams), C.c_void_p, C.c_void_p, C.c_int, dp, C.c_int]
        L.ora_das.restype = C.c_int
        L.ora_fir_taps.argtypes = [C.c_int, C.c_double, C.c_double, dp]
        L.ora_iq_envelope.argtypes = [dp, C.c_int, C.c_double, C.c_double, C.c_double, C.c_int,
                                      C.c_int, dp]
        L.ora_iq_envelope.restype = C.c_int
        L.ora_compound.argtypes = [dp, C.c_int, C.c_double, C.c_int, dp, dp, dp, C.c_int, C.c_int, dp]
        L.ora_compound.restype = C.c_int
        L.ora_log_compress.argtypes = [dp, C.c_long, C.c_int, C.c_double, C.c_double, dp]
        L.ora_log_compress.restype = C.c_double
        L.ora_to_u8.argtypes = [dp, C.c_long, C.c_void_p]
        L.ora_sc_table.argtypes = [C.POINTER(_ScParams), C.c_void_p, C.c_void_p, dp]
        L.ora_scan_convert.argtypes = [C.POINTER(_ScParams), dp, dp, C.c_void_p]
        _lib = L
    return _lib


def _dptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def element_positions(nx, ny, px, py):
    pos = np.zeros((nx * ny, 3), np.float64)
    lib().ora_element_positions(nx, ny, px, py, _dptr(pos))
    return pos


def dr_mm(c_mps, fs_hz):
    return lib().ora_dr_mm(c_mps, fs_hz)


def delay_samples(origin, direction, elem, z_mm, fs_hz, c_mps, t0_s=0.0):
    o = np.ascontiguousarray(origin, np.float64)
    d = np.ascontiguousarray(direction, np.float64)
    e = np.ascontiguousarray(elem, np.float64)
    return lib().ora_delay_samples(_dptr(o), _dptr(d), _dptr(e), z_mm, fs_hz, c_mps, t0_s)


def das(cfg, raw, lines=None, nthreads=None):
    """RF [nlines][S] (float64) for one frame raw [E][C][S] int16.

    ``cfg`` is a ``synth.configs.Workload`` (or any object with the same
    attributes); ``lines`` selects a subset of scanlines (default: all)."""
    raw = np.ascontiguousarray(raw, np.int16)
    E, Cc, S = raw.shape
    chmap = getattr(cfg, "channel_element", None)
    nch = 0 if chmap is None else int(np.shape(chmap)[1])
    chmap = None if chmap is None else np.ascontiguousarray(chmap, np.int32)
    assert E == cfg.num_events and S == cfg.S
    assert Cc == (nch if nch else cfg.elements_x * cfg.elements_y)
    org = np.ascontiguousarray(cfg.line_origin_mm, np.float64)
    dirs = np.ascontiguousarray(cfg.line_direction, np.float64)
    ev = np.ascontiguousarray(cfg.line_event, np.int32)
    L = org.shape[0]
    if lines is None:
        lines = np.arange(L, dtype=np.int32)
    lines = np.ascontiguousarray(lines, np.int32)
    p = _DasParams(cfg.elements_x, cfg.elements_y, cfg.pitch_x_mm, cfg.pitch_y_mm, E, S,
                   cfg.fs_hz, cfg.c_mps, cfg.t0_s, L, _dptr(org), _dptr(dirs),
                   ev.ctypes.data_as(C.POINTER(C.c_int32)), cfg.f_number, cfg.window,
                   cfg.normalize, nch,
                   None if chmap is None else chmap.ctypes.data_as(C.POINTER(C.c_int32)),
                   int(getattr(cfg, "interpolation", 0)))
    rf = np.zeros((len(lines), S), np.float64)
    nt = nthreads or min(len(lines), os.cpu_count() or 1)
    rc = lib().ora_das(C.byref(p), raw.ctypes.data, lines.ctypes.data, len(lines), _dptr(rf),
                       max(1, nt))
    assert rc == 0
    return rf


def fir_taps(T, fc_hz, fs_hz):
    h = np.zeros(T, np.float64)
    lib().ora_fir_taps(T, fc_hz, fs_hz, _dptr(h))
    return h


def iq_envelope(rf, fs_hz, fd_hz, bw_hz, taps=65, decimation=1):
    """Envelope per line, rf [..., S] -> [..., S//decimation] (float64)."""
    rf = np.ascontiguousarray(rf, np.float64)
    shp = rf.shape
    S = shp[-1]
    flat = rf.reshape(-1, S)
    out = np.zeros((flat.shape[0], S // decimation), np.float64)
    for i in range(flat.shape[0]):
        row = np.ascontiguousarray(flat[i])
        o = np.zeros(S // decimation, np.float64)
        rc = lib().ora_iq_envelope(_dptr(row), S, fs_hz, fd_hz, bw_hz, taps, decimation, _dptr(o))
        assert rc == 0
        out[i] = o
    return out.reshape(shp[:-1] + (S // decimation,))


def compound(rf, fs_hz, bands, taps=65, decimation=1):
    """Frequency-compounded envelope: sum_b w_b * IQ envelope
    of band b, bands = ((center Hz, bandwidth Hz, weight), ...); rf [..., S]."""
    rf = np.ascontiguousarray(rf, np.float64)
    shp = rf.shape
    S = shp[-1]
    flat = rf.reshape(-1, S)
    fd = np.ascontiguousarray([b[0] for b in bands], np.float64)
    bw = np.ascontiguousarray([b[1] for b in bands], np.float64)
    wt = np.ascontiguousarray([b[2] for b in bands], np.float64)
    out = np.zeros((flat.shape[0], S // decimation), np.float64)
    for i in range(flat.shape[0]):
        row = np.ascontiguousarray(flat[i])
        o = np.zeros(S // decimation, np.float64)
        rc = lib().ora_compound(_dptr(row), S, fs_hz, len(bands), _dptr(fd), _dptr(bw), _dptr(wt),
                                taps, decimation, _dptr(o))
        assert rc == 0
        out[i] = o
    return out.reshape(shp[:-1] + (S // decimation,))


def envelope(cfg, rf):
    """The envelope step a workload configures: compounding when cfg.bands is
    set, else the single IQ band (demod_frequency, demod_bandwidth)."""
    if getattr(cfg, "bands", ()):
        return compound(rf, cfg.fs_hz, cfg.bands, cfg.fir_taps, cfg.decimation)
    return iq_envelope(rf, cfg.fs_hz, cfg.demod_frequency_hz, cfg.demod_bandwidth_hz,
                       cfg.fir_taps, cfg.decimation)


def hilbert_envelope(x):
    """|analytic signal| by the DFT method: zero negative
    frequencies, double positive ones, keep DC and Nyquist, inverse DFT,
    modulus.  numpy.fft is the library step."""
    x = np.asarray(x, np.float64)
    N = x.shape[-1]
    X = np.fft.fft(x, axis=-1)
    g = np.zeros(N)
    g[0] = 1.0
    if N % 2 == 0:
        g[N // 2] = 1.0
        g[1:N // 2] = 2.0
    else:
        g[1:(N + 1) // 2] = 2.0
    return np.abs(np.fft.ifft(X * g, axis=-1))


def log_compress(env, dynamic_range_db=50.0, ref_mode=0, ref_value=1.0):
    """(y, ref) with y = clamp((20 log10(x/ref) + DR)/DR, 0, 1) over the whole
    array (one frame)."""
    x = np.ascontiguousarray(env, np.float64)
    y = np.zeros_like(x)
    ref = lib().ora_log_compress(_dptr(x), x.size, ref_mode, ref_value, dynamic_range_db,
                                 _dptr(y))
    return y, ref


def to_u8(y):
    y = np.ascontiguousarray(y, np.float64)
    out = np.zeros(y.shape, np.uint8)
    lib().ora_to_u8(_dptr(y), y.size, out.ctypes.data)
    return out


def _sc_params(cfg):
    o = np.asarray(cfg.line_origin_mm, np.float64)
    # the line image holds S // d samples spaced d * dr (decimation d)
    d = int(getattr(cfg, "decimation", 1))
    return _ScParams(cfg.sc_kind, cfg.num_lines_x, cfg.num_lines_y, cfg.S // d,
                     dr_mm(cfg.c_mps, cfg.fs_hz) * d, float(o[0, 0]), float(o[-1, 0]),
                     cfg.fov_x_deg, cfg.fov_y_deg, cfg.out_dims[0], cfg.out_dims[1],
                     cfg.out_dims[2], (C.c_double * 3)(*cfg.out_origin_mm),
                     (C.c_double * 3)(*cfg.out_spacing_mm))


def sc_table(cfg):
    """(valid [n] u8, idx [n,3] int32 (i0x, i0y, k0), frac [n,3] f64), n = nz*ny*nx."""
    p = _sc_params(cfg)
    n = cfg.out_dims[0] * cfg.out_dims[1] * cfg.out_dims[2]
    valid = np.zeros(n, np.uint8)
    idx = np.zeros((n, 3), np.int32)
    frac = np.zeros((n, 3), np.float64)
    lib().ora_sc_table(C.byref(p), valid.ctypes.data, idx.ctypes.data, _dptr(frac))
    return valid, idx, frac


def scan_convert(cfg, line_img):
    """(img [nz, ny, nx] f64, mask u8) from the log-compressed line image of
    one frame, line_img [Ly*Lx][S]."""
    p = _sc_params(cfg)
    li = np.ascontiguousarray(line_img, np.float64)
    nx, ny, nz = cfg.out_dims
    img = np.zeros((nz, ny, nx), np.float64)
    mask = np.zeros((nz, ny, nx), np.uint8)
    lib().ora_scan_convert(C.byref(p), _dptr(li), _dptr(img), mask.ctypes.data)
    return img, mask


def bmode_frame(cfg, raw, nthreads=None):
    """Whole oracle chain for one frame: (rf, env, y_line, ref)."""
    rf = das(cfg, raw, nthreads=nthreads)
    env = envelope(cfg, rf)
    y, ref = log_compress(env, cfg.dynamic_range_db, cfg.reference_mode, cfg.reference_value)
    return rf, env, y, ref
