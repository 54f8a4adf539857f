"""Workload definitions C1-C5 -- seeded, synthetic.

INPUT GENERATION ONLY.  This module builds the geometry arrays every
``supra_bf_config`` field needs (element grid, scanline origins/directions,
line->event map, output grid) and the scatterer recipes.  It holds none of
the method's arithmetic (no delay-and-sum, envelope, compression or scan
conversion); both the oracle and the CUDA path consume what it produces.

Units follow SPEC: mm, Hz, m/s, s, degrees.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

WIN_RECT, WIN_HANN, WIN_HAMMING = 0, 1, 2
INTERP_LINEAR, INTERP_NEAREST = 0, 1
NORM_COUNT, NORM_NONE = 0, 1
REF_FRAME_MAX, REF_FIXED = 0, 1
T_I16, T_F32, T_U8 = 0, 1, 2
SC_LINEAR_2D, SC_SECTOR_2D, SC_PYRAMID_3D = 0, 1, 2

C_MPS = 1540.0          # S:87 (the paper never states c)
FS_HZ = 40e6            # reading #1 (the paper never states fs)


def dr_mm(c_mps: float = C_MPS, fs_hz: float = FS_HZ) -> float:
    """Depth per sample c/(2 fs) in mm -- used here only to place
    synthetic scatterers and size output grids."""
    return 1000.0 * c_mps / (2.0 * fs_hz)


@dataclasses.dataclass
class Workload:
    name: str
    elements_x: int
    elements_y: int
    pitch_x_mm: float
    pitch_y_mm: float
    center_frequency_hz: float
    num_events: int
    S: int
    num_lines_x: int
    num_lines_y: int
    line_origin_mm: np.ndarray      # [L][3]
    line_direction: np.ndarray      # [L][3]
    line_event: np.ndarray          # [L] int32
    tx_origin_mm: np.ndarray        # [E][3] transmit reference per event (synth only)
    sc_kind: int
    out_dims: tuple                 # (nx, ny, nz)
    out_origin_mm: tuple
    out_spacing_mm: tuple
    fov_x_deg: float = 0.0
    fov_y_deg: float = 0.0
    fs_hz: float = FS_HZ
    c_mps: float = C_MPS
    t0_s: float = 0.0
    f_number: float = 1.0
    window: int = WIN_HANN
    normalize: int = NORM_COUNT
    demod_frequency_hz: float = 0.0     # default: f0
    demod_bandwidth_hz: float = 0.0     # default: 0.6 f0
    fir_taps: int = 65
    decimation: int = 1
    # frequency compounding: ((center Hz, bandwidth Hz,
    # weight), ...); empty = the single (demod_frequency, demod_bandwidth) band
    bands: tuple = ()
    # receive channel map [E][channels] -> element (-1 unused); None = one
    # channel per element ("only 64 channels usable")
    channel_element: Optional[np.ndarray] = None
    # fractional-delay lookup: 0 linear, 1 nearest (reading #32)
    interpolation: int = 0
    dynamic_range_db: float = 50.0
    reference_mode: int = REF_FRAME_MAX
    reference_value: float = 1.0
    line_output_type: int = T_F32
    sc_output_type: int = T_F32
    frames: int = 1                     # frames in the stream this config names
    realisations: int = 1               # distinct synthetic realisations cycled
    pulse_fbw: float = 0.3              # reading #27
    noise_db: Optional[float] = None    # white noise re max, None = off
    seed: int = 0

    def __post_init__(self):
        if self.demod_frequency_hz == 0.0:
            self.demod_frequency_hz = self.center_frequency_hz
        if self.demod_bandwidth_hz == 0.0:
            self.demod_bandwidth_hz = 0.6 * self.center_frequency_hz
        self.line_origin_mm = np.ascontiguousarray(self.line_origin_mm, np.float64)
        self.line_direction = np.ascontiguousarray(self.line_direction, np.float64)
        self.line_event = np.ascontiguousarray(self.line_event, np.int32)
        self.tx_origin_mm = np.ascontiguousarray(self.tx_origin_mm, np.float64)

    @property
    def L(self) -> int:
        return self.num_lines_x * self.num_lines_y

    @property
    def C(self) -> int:
        """Traces per event in the raw frame."""
        if self.channel_element is not None:
            return int(np.shape(self.channel_element)[1])
        return self.elements_x * self.elements_y

    @property
    def out_pixels(self) -> int:
        return self.out_dims[0] * self.out_dims[1] * self.out_dims[2]

    def replace(self, **kw) -> "Workload":
        return dataclasses.replace(self, **kw)

    def raw_bytes_per_frame(self) -> int:
        return self.num_events * self.C * self.S * 2


# ---------------------------------------------------------------- geometry
def element_x(n: int, pitch: float) -> np.ndarray:
    return (np.arange(n) - (n - 1) / 2.0) * pitch


def linear_lines(xs: np.ndarray):
    L = len(xs)
    o = np.zeros((L, 3))
    o[:, 0] = xs
    d = np.zeros((L, 3))
    d[:, 2] = 1.0
    return o, d


def angle_grid_rad(n: int, fov_deg: float) -> np.ndarray:
    """theta_i = (i - (n-1)/2) * fov/(n-1) (reading #14)."""
    if n == 1:
        return np.zeros(1)
    fov = fov_deg * math.pi / 180.0
    return (np.arange(n) - (n - 1) / 2.0) * (fov / (n - 1))


def phased_lines(nx: int, fov_x_deg: float, ny: int = 1, fov_y_deg: float = 0.0):
    """Directions d = (sin tx, cos tx sin ty, cos tx cos ty), origin 0
    (reading #13); line l = ly*nx + lx."""
    tx = angle_grid_rad(nx, fov_x_deg)
    ty = angle_grid_rad(ny, fov_y_deg) if ny > 1 else np.zeros(1)
    TY, TX = np.meshgrid(ty, tx, indexing="ij")
    d = np.stack([np.sin(TX), np.cos(TX) * np.sin(TY), np.cos(TX) * np.cos(TY)], -1).reshape(-1, 3)
    o = np.zeros_like(d)
    return o, d


def tx_origins(line_origin: np.ndarray, line_event: np.ndarray, E: int) -> np.ndarray:
    out = np.zeros((E, 3))
    for e in range(E):
        out[e] = line_origin[line_event == e].mean(0)
    return out


# ---------------------------------------------------------------- configs
def c1(**kw) -> Workload:
    """C1 parity/focus: linear 64 el, 0.3 mm, 7 MHz; 64 lines at the
    element centres; E=64, S=1024, 1 frame; one point at (x_32, 0, 600 dr)."""
    xs = element_x(64, 0.3)
    o, d = linear_lines(xs)
    ev = np.arange(64, dtype=np.int32)
    s = 0.0225
    w = Workload("C1", 64, 1, 0.3, 0.3, 7e6, 64, 1024, 64, 1, o, d, ev, tx_origins(o, ev, 64),
                 SC_LINEAR_2D, (841, 1, 876), (-9.45, 0.0, 0.0), (s, s, s))
    return w.replace(**kw) if kw else w


def c2(variant: str = "a", **kw) -> Workload:
    """C2 2D stream: linear 128 el, 256 lines over the element span, S=2048,
    100 frames cycling 4 speckle realisations.  Variant 'b': E=128, M=2 block
    multi-line (ev = l // 2)."""
    xs = -19.05 + np.arange(256) * (38.1 / 255)
    o, d = linear_lines(xs)
    if variant == "b":
        E, ev = 128, (np.arange(256) // 2).astype(np.int32)
    else:
        E, ev = 256, np.arange(256, dtype=np.int32)
    s = 0.0225
    w = Workload("C2" + ("b" if variant == "b" else ""), 128, 1, 0.3, 0.3, 7e6, E, 2048, 256, 1,
                 o, d, ev, tx_origins(o, ev, E), SC_LINEAR_2D, (1694, 1, 1752),
                 (-19.05, 0.0, 0.0), (s, s, s), frames=100, realisations=4, noise_db=-60.0)
    return w.replace(**kw) if kw else w


def c3(**kw) -> Workload:
    """C3 sector: phased 128 el, 0.22 mm, 3.5 MHz; 192 lines over 60 deg;
    S=4096; sector scan conversion to 512 x 512."""
    o, d = phased_lines(192, 60.0)
    ev = np.arange(192, dtype=np.int32)
    S = 4096
    sp = (S - 1) * dr_mm() / 511
    w = Workload("C3", 128, 1, 0.22, 0.22, 3.5e6, 192, S, 192, 1, o, d, ev, tx_origins(o, ev, 192),
                 SC_SECTOR_2D, (512, 1, 512), (-255.5 * sp, 0.0, 0.0), (sp, sp, sp),
                 fov_x_deg=60.0, frames=16, noise_db=-60.0, seed=10)
    return w.replace(**kw) if kw else w


def c4(variant: str = "b", **kw) -> Workload:
    """C4 3D: matrix 32 x 32, 0.3 mm, 7 MHz; 64 x 64 lines over
    60 x 60 deg; S=2048; pyramid scan conversion to 256^3.  Variant 'a':
    E=4096, M=1; 'b': E=256, 4x4 block multi-line (reading #24)."""
    o, d = phased_lines(64, 60.0, 64, 60.0)
    lx = np.tile(np.arange(64), 64)
    ly = np.repeat(np.arange(64), 64)
    if variant == "a":
        E, ev = 4096, np.arange(4096, dtype=np.int32)
    else:
        E, ev = 256, ((lx // 4) * 16 + ly // 4).astype(np.int32)
    S = 2048
    sp = (S - 1) * dr_mm() / 255
    w = Workload("C4" + variant, 32, 32, 0.3, 0.3, 7e6, E, S, 64, 64, o, d, ev,
                 tx_origins(o, ev, E), SC_PYRAMID_3D, (256, 256, 256),
                 (-127.5 * sp, -127.5 * sp, 0.0), (sp, sp, sp), fov_x_deg=60.0, fov_y_deg=60.0,
                 noise_db=-40.0)
    return w.replace(**kw) if kw else w


def walking_aperture(n_elements: int, n_channels: int, pitch_mm: float,
                     tx_x_mm: np.ndarray) -> np.ndarray:
    """Receive channel map of a walking (sliding) active aperture (the
    128-element probe with 64 usable channels; S:102 leaves the policy open,
    reading #31): event e records the n_channels contiguous elements whose
    centre is nearest its transmit position, clamped to the array;
    channel ch -> element a0(e) + ch.  [E][n_channels] int32."""
    x0 = -(n_elements - 1) / 2.0 * pitch_mm
    a0 = np.rint((np.asarray(tx_x_mm) - x0) / pitch_mm - (n_channels - 1) / 2.0).astype(np.int64)
    a0 = np.clip(a0, 0, n_elements - n_channels)
    return (a0[:, None] + np.arange(n_channels)[None, :]).astype(np.int32)


def table1(tx_events: int = 128, multiline: int = 2, frames: int = 1, **kw) -> Workload:
    """The paper's 2D benchmark shapes, Table 1 "(a / b)" = (transmit events /
    multi-line factor): CPLA12875 linear probe, 128 elements,
    0.3 mm pitch, 7 MHz, 64 usable receive channels (walking aperture), depth
    45 mm (S = 2368 samples = 45.6 mm at 40 MHz, a multiple of 32),
    interleaved multi-line: tx_events * M - (M - 1) lines, line l ->
    event floor(l / M), origins evenly spaced over the element span
    (S:53); scan conversion on the paper's 0.0225 mm grid."""
    E, M = tx_events, multiline
    ev = interleaved_line_events(E, M)
    L = len(ev)
    xs = -19.05 + np.arange(L) * (38.1 / (L - 1))
    o, d = linear_lines(xs)
    tx = tx_origins(o, ev, E)
    chm = walking_aperture(128, 64, 0.3, tx[:, 0])
    s = 0.0225
    S = 2368
    nz = int(math.floor(45.0 / s)) + 1                   # 0 .. 45 mm
    w = Workload(f"T1_{E}_{M}", 128, 1, 0.3, 0.3, 7e6, E, S, L, 1, o, d, ev, tx,
                 SC_LINEAR_2D, (1694, 1, nz), (-19.05, 0.0, 0.0), (s, s, s), frames=frames,
                 realisations=min(4, max(1, frames)), noise_db=-60.0, channel_element=chm)
    return w.replace(**kw) if kw else w


def c4p(volumes: int = 1, **kw) -> Workload:
    """The paper's own 3D row:
    32 x 32 matrix probe (0.3 mm, 7 MHz) driven through 384 channels,
    32 x 16 = 512 scanlines over a 60 x 60 deg field of view, 70 mm depth
    (S = 3648 samples = 70.2 mm at 40 MHz, a multiple of 32), one transmit
    per line; 0.175 mm isotropic pyramid scan conversion (401 x 401 x 402).
    The 384 channels are the 12 central element rows (j = 10 .. 21, all 32
    columns) for every event (reading #33: the paper does not say which
    elements its 384-channel system drives)."""
    o, d = phased_lines(32, 60.0, 16, 60.0)
    E = 512
    ev = np.arange(E, dtype=np.int32)
    S = 3648
    chm = np.tile((10 * 32 + np.arange(384)).astype(np.int32), (E, 1))
    sp = 0.175
    rmax = (S - 1) * dr_mm()
    half = int(math.floor(rmax * math.sin(math.radians(30.0)) / sp))
    nz = int(math.floor(rmax / sp)) + 1
    w = Workload("C4p", 32, 32, 0.3, 0.3, 7e6, E, S, 32, 16, o, d, ev, tx_origins(o, ev, E),
                 SC_PYRAMID_3D, (2 * half + 1, 2 * half + 1, nz), (-half * sp, -half * sp, 0.0),
                 (sp, sp, sp), fov_x_deg=60.0, fov_y_deg=60.0, noise_db=-40.0, frames=volumes,
                 channel_element=chm)
    return w.replace(**kw) if kw else w


def wire_phantom(depths_mm, x_mm=0.0, reflectivity=1.0) -> np.ndarray:
    """SPEC wire_phantom (the paper's water-tank wire target at
    5, 10, 15, 20, 25 mm): one unit-reflectivity scatterer per
    depth, centred laterally.  [n][4] = (x, y, z, reflectivity)."""
    d = np.asarray(list(depths_mm), np.float64)
    out = np.zeros((len(d), 4))
    out[:, 0], out[:, 2], out[:, 3] = x_mm, d, reflectivity
    return out


def psf_linear(half_width_mm: float = 3.0, n_lines: int = 201, S: int = 1408, **kw) -> Workload:
    """PSF measurement layout (f3; Fig. 4): the 128-element 0.3 mm
    7 MHz linear probe with all 128 channels, ``n_lines`` lines
    evenly spaced over +-half_width_mm around the array centre (dense
    lateral sampling, 0.03 mm for the default), one transmit per line from
    the line origin, S samples (27.1 mm for the default)."""
    xs = np.linspace(-half_width_mm, half_width_mm, n_lines)
    o, d = linear_lines(xs)
    ev = np.arange(n_lines, dtype=np.int32)
    s = 0.0225
    nx = int(round(2 * half_width_mm / s)) + 1
    nz = int(math.floor((S - 1) * dr_mm() / s)) + 1
    w = Workload("PSF", 128, 1, 0.3, 0.3, 7e6, n_lines, S, n_lines, 1, o, d, ev, tx_origins(o, ev, n_lines),
                 SC_LINEAR_2D, (nx, 1, nz), (-half_width_mm, 0.0, 0.0), (s, s, s))
    return w.replace(**kw) if kw else w


CONFIGS = {"C1": c1, "C2": c2, "C3": c3, "C4a": lambda **k: c4("a", **k),
           "C4b": lambda **k: c4("b", **k), "C2b": lambda **k: c2("b", **k),
           "T1_64_1": lambda **k: table1(64, 1, **k), "T1_64_2": lambda **k: table1(64, 2, **k),
           "T1_128_1": lambda **k: table1(128, 1, **k), "T1_128_2": lambda **k: table1(128, 2, **k),
           "C4p": c4p}


# ------------------------------------------------------------- scatterers
def scatterers(w: Workload, realisation: int = 0) -> np.ndarray:
    """[n][4] = (x, y, z, reflectivity) in mm, seeded (NumPy PCG64)."""
    name = w.name
    if name == "C1":
        return np.array([[0.15, 0.0, 600 * dr_mm(w.c_mps, w.fs_hz), 1.0]])
    rng = np.random.Generator(np.random.PCG64(w.seed + realisation))
    if name.startswith("T1_"):
        # Table-1 phantom: speckle over the 38.1 x 45 mm field + 3 wires
        n = 20000
        x = rng.uniform(-19.05, 19.05, n)
        z = rng.uniform(1.0, 44.0, n)
        s = np.zeros((n + 3, 4))
        s[:n, 0], s[:n, 2], s[:n, 3] = x, z, rng.standard_normal(n)
        s[n:] = [[-8, 0, 12, 20], [0, 0, 25, 20], [8, 0, 38, 20]]
        return s
    if name.startswith("C2"):
        n = 20000
        pts = []
        while sum(len(p) for p in pts) < n:
            x = rng.uniform(-19.05, 19.05, n)
            z = rng.uniform(1.0, 39.0, n)
            keep = (x ** 2 + (z - 20.0) ** 2) > 16.0      # 4 mm anechoic cyst
            pts.append(np.stack([x[keep], z[keep]], 1))
        xz = np.concatenate(pts)[:n]
        refl = rng.standard_normal(n)
        s = np.zeros((n + 3, 4))
        s[:n, 0], s[:n, 2], s[:n, 3] = xz[:, 0], xz[:, 1], refl
        s[n:] = [[-10, 0, 10, 20], [0, 0, 30, 20], [10, 0, 15, 20]]
        return s
    if name == "C3":
        n = 20000
        r = rng.uniform(2.0, 78.0, n)
        th = rng.uniform(-math.pi / 6, math.pi / 6, n)
        refl = rng.standard_normal(n)
        s = np.zeros((n + 7, 4))
        s[:n, 0], s[:n, 2], s[:n, 3] = r * np.sin(th), r * np.cos(th), refl
        for i, zz in enumerate(range(10, 80, 10)):
            s[n + i] = [0, 0, zz, 20]
        return s
    if name == "C4p":
        # wire grid over the paper's 70 mm pyramid
        pts = []
        for tx in (-20, 0, 20):
            for ty in (-20, 0, 20):
                for r in (10, 25, 40, 55, 68):
                    a, b = math.radians(tx), math.radians(ty)
                    pts.append([r * math.sin(a), r * math.cos(a) * math.sin(b),
                                r * math.cos(a) * math.cos(b), 1.0])
        return np.array(pts)
    if name.startswith("C4"):
        pts = []
        for tx in (-20, -10, 0, 10, 20):
            for ty in (-20, -10, 0, 10, 20):
                for r in (8, 14, 20, 26, 32):
                    a, b = math.radians(tx), math.radians(ty)
                    pts.append([r * math.sin(a), r * math.cos(a) * math.sin(b),
                                r * math.cos(a) * math.cos(b), 1.0])
        return np.array(pts)
    raise KeyError(name)


def interleaved_line_events(E: int, M: int) -> np.ndarray:
    """Interleaved multi-line layout: E*M - (M-1) receive
    lines, transmit lines at every M-th position, line l -> event floor(l/M)."""
    L = E * M - (M - 1)
    return (np.arange(L) // M).astype(np.int32)
