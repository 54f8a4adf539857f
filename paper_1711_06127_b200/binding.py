"""Thin ctypes binding over libsupra_bf.so (include/supra_bf.h).

Argument marshalling only: every step of the hot path runs in the library's
sm_100a kernels.  Tensors are torch CUDA tensors (device memory, streams);
there is no CPU fallback -- if the shared library or a CUDA device is
missing, construction raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# The in-tree build.  No environment variable selects another library: a
# dev script that A/B-times a variant build calls use_library() explicitly.
LIB_PATH = os.path.join(HERE, "libsupra_bf.so")

ABI_VERSION = 2
MAX_BANDS = 4
OK, E_PARAM, E_STRUCT, E_RESOURCE, E_CUDA = 0, 2, 3, 4, 5
WIN_RECT, WIN_HANN, WIN_HAMMING = 0, 1, 2
INTERP_LINEAR, INTERP_NEAREST = 0, 1
NORM_COUNT, NORM_NONE = 0, 1
REF_FRAME_MAX, REF_FIXED = 0, 1
T_I16, T_F32, T_U8 = 0, 1, 2
SC_LINEAR_2D, SC_SECTOR_2D, SC_PYRAMID_3D = 0, 1, 2

EXPORTS = ("supra_bf_create", "supra_bf_beamform", "supra_bf_envelope_log", "supra_bf_scanconvert",
           "supra_bf_destroy", "supra_bf_last_error", "supra_bf_sc_indices", "supra_bf_info",
           "supra_bf_set_das_events", "supra_bf_beamform_lines", "supra_bf_log_compress",
           "supra_bf_beamform_bmode", "supra_bf_stage_raw")


class SupraError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"supra_bf status {status}: {msg}")
        self.status = status


class Config(C.Structure):
    """Mirror of ``supra_bf_config`` (include/supra_bf.h)."""
    _fields_ = [
        ("abi_version", C.c_int32), ("device", C.c_int32),
        ("elements_x", C.c_int32), ("elements_y", C.c_int32),
        ("pitch_x_mm", C.c_double), ("pitch_y_mm", C.c_double),
        ("center_frequency_hz", C.c_double),
        ("num_events", C.c_int32), ("samples_per_channel", C.c_int32),
        ("input_type", C.c_int32),
        ("sample_frequency_hz", C.c_double), ("speed_of_sound_mps", C.c_double),
        ("t0_s", C.c_double),
        ("num_lines_x", C.c_int32), ("num_lines_y", C.c_int32),
        ("line_origin_mm", C.POINTER(C.c_double)), ("line_direction", C.POINTER(C.c_double)),
        ("line_event", C.POINTER(C.c_int32)),
        ("f_number", C.c_double), ("window", C.c_int32), ("normalize", C.c_int32),
        ("demod_frequency_hz", C.c_double), ("demod_bandwidth_hz", C.c_double),
        ("fir_taps", C.c_int32), ("decimation", C.c_int32),
        ("dynamic_range_db", C.c_double), ("reference_value", C.c_double),
        ("reference_mode", C.c_int32), ("line_output_type", C.c_int32),
        ("sc_kind", C.c_int32), ("sc_output_type", C.c_int32),
        ("out_dims", C.c_int32 * 3),
        ("out_origin_mm", C.c_double * 3), ("out_spacing_mm", C.c_double * 3),
        ("fov_x_deg", C.c_double), ("fov_y_deg", C.c_double),
        ("max_frames_per_call", C.c_int32),
        ("num_bands", C.c_int32),
        ("band_center_hz", C.c_double * MAX_BANDS), ("band_bandwidth_hz", C.c_double * MAX_BANDS),
        ("band_weight", C.c_double * MAX_BANDS),
        ("num_channels", C.c_int32), ("channel_element", C.POINTER(C.c_int32)),
        ("interpolation", C.c_int32),
    ]


_lib = None


def lib():
    """Load libsupra_bf.so; raise if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_1711_06127_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        L.supra_bf_create.argtypes = [C.POINTER(Config), C.POINTER(vp)]
        L.supra_bf_create.restype = C.c_int
        L.supra_bf_beamform.argtypes = [vp, vp, C.c_int32, vp, vp, vp]
        L.supra_bf_beamform.restype = C.c_int
        L.supra_bf_envelope_log.argtypes = [vp, vp, C.c_int32, vp, vp]
        L.supra_bf_envelope_log.restype = C.c_int
        L.supra_bf_scanconvert.argtypes = [vp, vp, C.c_int32, vp, vp, vp]
        L.supra_bf_scanconvert.restype = C.c_int
        L.supra_bf_destroy.argtypes = [vp]
        L.supra_bf_destroy.restype = None
        L.supra_bf_last_error.argtypes = []
        L.supra_bf_last_error.restype = C.c_char_p
        L.supra_bf_sc_indices.argtypes = [vp, vp, vp]
        L.supra_bf_sc_indices.restype = C.c_int
        L.supra_bf_info.argtypes = [vp, vp]
        L.supra_bf_info.restype = C.c_int
        L.supra_bf_set_das_events.argtypes = [vp, vp, vp]
        L.supra_bf_set_das_events.restype = C.c_int
        L.supra_bf_beamform_lines.argtypes = [vp, vp, C.c_int32, C.c_int32, C.c_int32, vp, vp, vp]
        L.supra_bf_beamform_lines.restype = C.c_int
        L.supra_bf_log_compress.argtypes = [vp, vp, C.c_int32, C.c_int32, C.c_int32, vp, vp, vp]
        L.supra_bf_log_compress.restype = C.c_int
        L.supra_bf_beamform_bmode.argtypes = [vp, vp, C.c_int32, vp, vp, vp]
        L.supra_bf_beamform_bmode.restype = C.c_int
        L.supra_bf_stage_raw.argtypes = [vp, vp, vp, C.c_int32, vp, vp]
        L.supra_bf_stage_raw.restype = C.c_int
        _lib = L
    return _lib


def use_library(path: str):
    """Dev aid (scripts/ only): load another build of the same library, e.g.
    _variants/<name>/libsupra_bf.so, before the first handle is created."""
    global LIB_PATH
    if _lib is not None:
        raise RuntimeError("the library is already loaded")
    LIB_PATH = path


def _check(rc: int):
    if rc != OK:
        raise SupraError(rc, lib().supra_bf_last_error().decode())


def make_config(w, device: int = 0, max_frames: int = 1, **over) -> tuple:
    """Build a ``Config`` from a workload description (any object with the
    ``synth.configs.Workload`` attributes).  Returns (Config, keepalive)."""
    org = np.ascontiguousarray(w.line_origin_mm, np.float64)
    dirs = np.ascontiguousarray(w.line_direction, np.float64)
    ev = np.ascontiguousarray(w.line_event, np.int32)
    c = Config()
    c.abi_version = ABI_VERSION
    c.device = device
    c.elements_x, c.elements_y = w.elements_x, w.elements_y
    c.pitch_x_mm, c.pitch_y_mm = w.pitch_x_mm, w.pitch_y_mm
    c.center_frequency_hz = w.center_frequency_hz
    c.num_events, c.samples_per_channel, c.input_type = w.num_events, w.S, T_I16
    c.sample_frequency_hz, c.speed_of_sound_mps, c.t0_s = w.fs_hz, w.c_mps, w.t0_s
    c.num_lines_x, c.num_lines_y = w.num_lines_x, w.num_lines_y
    c.line_origin_mm = org.ctypes.data_as(C.POINTER(C.c_double))
    c.line_direction = dirs.ctypes.data_as(C.POINTER(C.c_double))
    c.line_event = ev.ctypes.data_as(C.POINTER(C.c_int32))
    c.f_number, c.window, c.normalize = w.f_number, w.window, w.normalize
    c.demod_frequency_hz, c.demod_bandwidth_hz = w.demod_frequency_hz, w.demod_bandwidth_hz
    c.fir_taps, c.decimation = w.fir_taps, w.decimation
    c.dynamic_range_db, c.reference_value = w.dynamic_range_db, w.reference_value
    c.reference_mode, c.line_output_type = w.reference_mode, w.line_output_type
    c.sc_kind, c.sc_output_type = w.sc_kind, w.sc_output_type
    c.out_dims = (C.c_int32 * 3)(*w.out_dims)
    c.out_origin_mm = (C.c_double * 3)(*w.out_origin_mm)
    c.out_spacing_mm = (C.c_double * 3)(*w.out_spacing_mm)
    c.fov_x_deg, c.fov_y_deg = w.fov_x_deg, w.fov_y_deg
    c.max_frames_per_call = max_frames
    bands = list(getattr(w, "bands", ()) or ())
    if len(bands) > MAX_BANDS:
        raise ValueError(f"at most {MAX_BANDS} compounding bands")
    c.num_bands = len(bands)
    for b, (fc, bw, wt) in enumerate(bands):
        c.band_center_hz[b], c.band_bandwidth_hz[b], c.band_weight[b] = fc, bw, wt
    c.interpolation = getattr(w, "interpolation", 0)
    chmap = getattr(w, "channel_element", None)
    if chmap is not None:
        chmap = np.ascontiguousarray(chmap, np.int32)
        c.num_channels = chmap.shape[1]
        c.channel_element = chmap.ctypes.data_as(C.POINTER(C.c_int32))
    for k, v in over.items():
        setattr(c, k, v)
    return c, (org, dirs, ev, chmap)


def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream(stream) -> Optional[int]:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


class SupraBF:
    """One handle = one configuration on one device (supra_bf_create)."""

    def __init__(self, w, device: int = 0, max_frames: int = 1, **over):
        self.w = w
        self.device = device
        self.cfg, keep = make_config(w, device, max_frames, **over)
        h = C.c_void_p()
        _check(lib().supra_bf_create(C.byref(self.cfg), C.byref(h)))
        del keep
        self.h = h
        self.L = w.num_lines_x * w.num_lines_y
        self.S = w.S
        self.Sd = w.S // max(1, w.decimation)   # line-image samples
        self.max_frames = max_frames

    # -- entry points ------------------------------------------------------
    def beamform(self, raw, frames: int, rf=None, line_img=None, stream=None):
        _check(lib().supra_bf_beamform(self.h, _ptr(raw), frames, _ptr(rf), _ptr(line_img),
                                       _stream(stream)))

    def envelope_log(self, rf, frames: int, line_img, stream=None):
        _check(lib().supra_bf_envelope_log(self.h, _ptr(rf), frames, _ptr(line_img),
                                           _stream(stream)))

    def beamform_lines(self, raw, frames: int, line_first: int, line_count: int, env, frame_max,
                       stream=None):
        """DAS + envelope for a line range; env f32 [F][L][S], frame_max f32 [F]."""
        _check(lib().supra_bf_beamform_lines(self.h, _ptr(raw), frames, line_first, line_count,
                                             _ptr(env), _ptr(frame_max), _stream(stream)))

    def log_compress(self, env, frames: int, line_first: int, line_count: int, frame_max, line_img,
                     stream=None):
        """Log compression of a line range against frame_max (or the fixed reference)."""
        _check(lib().supra_bf_log_compress(self.h, _ptr(env), frames, line_first, line_count,
                                           _ptr(frame_max), _ptr(line_img), _stream(stream)))

    def beamform_bmode(self, raw, frames: int, img, mask=None, stream=None):
        """raw -> B-mode in one call (DAS + envelope, log compression inside
        scan conversion); img as for scanconvert."""
        _check(lib().supra_bf_beamform_bmode(self.h, _ptr(raw), frames, _ptr(img), _ptr(mask),
                                             _stream(stream)))

    def stage_raw(self, src, dst, frames: int, stream=None) -> int:
        """Copy the referenced sample ranges of src (pinned host or device
        int16 [F][E][C][S]) into device dst; returns the bytes moved per frame."""
        n = C.c_int64(0)
        _check(lib().supra_bf_stage_raw(self.h, _ptr(src), _ptr(dst), frames, C.byref(n), _stream(stream)))
        return int(n.value)

    def scanconvert(self, line_img, frames: int, img, mask=None, stream=None):
        _check(lib().supra_bf_scanconvert(self.h, _ptr(line_img), frames, _ptr(img), _ptr(mask),
                                          _stream(stream)))

    def close(self):
        if getattr(self, "h", None):
            lib().supra_bf_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- introspection -----------------------------------------------------
    def info(self) -> dict:
        a = np.zeros(8, np.int64)
        _check(lib().supra_bf_info(self.h, a.ctypes.data))
        keys = ("kernels_per_beamform", "frames_per_cta", "tile_k", "referenced_bytes_per_frame",
                "taps_per_frame", "sc_table_bytes", "sc_valid_pixels", "kernels_per_scanconvert")
        return {k: int(v) for k, v in zip(keys, a)}

    def set_das_events(self, before=None, after=None):
        """Record torch.cuda.Event ``before``/``after`` around the DAS launch."""
        b = None if before is None else before.cuda_event
        a = None if after is None else after.cuda_event
        _check(lib().supra_bf_set_das_events(self.h, b, a))

    def sc_indices(self):
        n = int(np.prod(self.w.out_dims))
        valid = np.zeros(n, np.uint8)
        idx = np.zeros((n, 3), np.int32)
        _check(lib().supra_bf_sc_indices(self.h, valid.ctypes.data, idx.ctypes.data))
        return valid, idx

    # -- allocation helpers (torch device memory) ------------------------------
    def empty_line_img(self, frames: int):
        import torch
        dt = torch.uint8 if self.w.line_output_type == T_U8 else torch.float32
        return torch.empty((frames, self.L, self.Sd), dtype=dt, device=f"cuda:{self.device}")

    def empty_rf(self, frames: int):
        import torch
        return torch.empty((frames, self.L, self.S), dtype=torch.float32,
                           device=f"cuda:{self.device}")

    def empty_img(self, frames: int):
        import torch
        nx, ny, nz = self.w.out_dims
        dt = torch.uint8 if self.w.sc_output_type == T_U8 else torch.float32
        return torch.empty((frames, nz, ny, nx), dtype=dt, device=f"cuda:{self.device}")

    def empty_mask(self):
        import torch
        nx, ny, nz = self.w.out_dims
        return torch.empty((nz, ny, nx), dtype=torch.uint8, device=f"cuda:{self.device}")
