"""Point-spread-function measurement (SPEC measure_psf; the
paper's wire-target evaluation, Fig. 4): locate the peak of a
pre-log amplitude image, take the lateral and axial profiles through it and
report the full width at half maximum, each side found by linear
interpolation of the profile where it crosses half the peak.  Test/analysis
support only (not part of the product path)."""
from __future__ import annotations

import numpy as np


def fwhm(profile, spacing: float, ipk: int | None = None) -> float:
    """FWHM (same unit as ``spacing``) of a 1-D amplitude profile around its
    peak (index ``ipk``, default argmax); NaN when a side never falls below
    half (peak at the boundary: flagged)."""
    p = np.asarray(profile, np.float64)
    i = int(np.argmax(p)) if ipk is None else int(ipk)
    half = 0.5 * p[i]
    # right crossing
    r = i
    while r + 1 < len(p) and p[r + 1] > half:
        r += 1
    if r + 1 >= len(p):
        return float("nan")
    xr = r + (p[r] - half) / (p[r] - p[r + 1])
    lft = i
    while lft - 1 >= 0 and p[lft - 1] > half:
        lft -= 1
    if lft - 1 < 0:
        return float("nan")
    xl = lft - (p[lft] - half) / (p[lft] - p[lft - 1])
    return float((xr - xl) * spacing)


def measure_psf(img, lateral_spacing: float, axial_spacing: float, expected_depth: float,
                lateral_origin: float = 0.0, depth_window: float = 2.0):
    """img [lateral][depth] pre-log amplitudes on a uniform grid (depth 0 at
    index 0).  The dominant peak within +-depth_window of expected_depth
    (S:529).  Returns dict(lateral_fwhm, axial_fwhm, peak_lateral, peak_depth)."""
    a = np.asarray(img, np.float64)
    k0 = max(0, int(np.floor((expected_depth - depth_window) / axial_spacing)))
    k1 = min(a.shape[1], int(np.ceil((expected_depth + depth_window) / axial_spacing)) + 1)
    sub = a[:, k0:k1]
    il, ik = np.unravel_index(int(np.argmax(sub)), sub.shape)
    ik += k0
    return {"lateral_fwhm": fwhm(a[:, ik], lateral_spacing, il),
            "axial_fwhm": fwhm(a[il, :], axial_spacing, ik),
            "peak_lateral": lateral_origin + il * lateral_spacing,
            "peak_depth": ik * axial_spacing}
