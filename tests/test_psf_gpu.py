"""End-to-end focusing quality on the GPU path: a synthetic
wire phantom at the paper's depths 5..25 mm (SPEC wire_phantom
S:441-446) through synth -> supra_bf_beamform_lines (DAS + IQ envelope,
pre-log) -> PSF/FWHM measurement (Fig. 4).  The paper's absolute
FWHM values are hardware-specific and not matched (parity unpinned there);
these are the SPEC's property checks."""
import math

import numpy as np
import pytest

import synth
from synth import configs
from psf import measure_psf

pytestmark = pytest.mark.gpu
DEPTHS = (5.0, 10.0, 15.0, 20.0, 25.0)


def _envelope(w, scat):
    import torch
    from paper_1711_06127_b200 import SupraBF
    raw = torch.empty((1, w.num_events, w.C, w.S), dtype=torch.int16, device="cuda")
    synth.channel_data_gpu(w, raw[0], scat=scat)
    bf = SupraBF(w)
    env = torch.zeros((1, w.L, w.S), dtype=torch.float32, device="cuda")
    fmax = torch.zeros((1,), dtype=torch.float32, device="cuda")
    bf.beamform_lines(raw, 1, 0, w.L, env, fmax)
    torch.cuda.synchronize()
    bf.close()
    return env[0].cpu().numpy().astype(np.float64)


def _sweep(w):
    env = _envelope(w, configs.wire_phantom(DEPTHS))
    dx = w.line_origin_mm[1, 0] - w.line_origin_mm[0, 0]
    dr = configs.dr_mm()
    return [measure_psf(env, dx, dr, z, lateral_origin=w.line_origin_mm[0, 0], depth_window=1.5)
            for z in DEPTHS]


def test_wire_phantom_psf_sweep_constant_f_number():
    w = configs.psf_linear()
    rep = _sweep(w)
    dr = configs.dr_mm()
    dx = w.line_origin_mm[1, 0] - w.line_origin_mm[0, 0]
    sig = synth.syn_sigma_samples(w.fs_hz, w.center_frequency_hz, w.pulse_fbw) if hasattr(
        synth, "syn_sigma_samples") else w.fs_hz / (2 * math.pi * w.pulse_fbw * w.center_frequency_hz
                                                    / (2 * math.sqrt(2 * math.log(2))))
    axial_expect = 2 * math.sqrt(2 * math.log(2)) * sig * dr      # c tau / 2 of the pulse envelope
    for z, r in zip(DEPTHS, rep):
        # echo timing: peak within +-1 depth sample and on the axis
        assert abs(r["peak_depth"] - z) <= dr + 1e-9, (z, r)
        assert abs(r["peak_lateral"]) <= dx + 1e-9, (z, r)
        # axial FWHM within 25 % of c tau / 2
        assert abs(r["axial_fwhm"] - axial_expect) <= 0.25 * axial_expect, (z, r, axial_expect)
        assert 0 < r["lateral_fwhm"] < 2.0
    # constant F-number: lateral FWHM within 30 % across 10..25 mm
    lat = np.array([r["lateral_fwhm"] for r in rep[1:]])
    assert lat.max() <= 1.3 * lat.min(), lat


def test_wire_phantom_fixed_aperture_lateral_fwhm_nondecreasing():
    # a tiny F-number opens the whole 128-element aperture at every depth
    # (fixed aperture): lateral FWHM non-decreasing with depth
    w = configs.psf_linear(f_number=0.02)
    lat = [r["lateral_fwhm"] for r in _sweep(w)]
    assert all(b >= a - 1e-3 for a, b in zip(lat, lat[1:])), lat


def test_two_wires_amplitude_ratio_S436():
    # reflectivities 1 and 0.5 at the same depth, well separated: envelope
    # peaks in ratio 0.5 +- 5 % (end-to-end linearity)
    w = configs.psf_linear(half_width_mm=4.0, n_lines=161)
    scat = np.concatenate([configs.wire_phantom([15.0], x_mm=-2.0, reflectivity=1.0),
                           configs.wire_phantom([15.0], x_mm=2.0, reflectivity=0.5)])
    env = _envelope(w, scat)
    x = w.line_origin_mm[:, 0]
    a = env[x < 0].max()
    b = env[x > 0].max()
    assert abs(b / a - 0.5) <= 0.05 * 0.5, b / a
