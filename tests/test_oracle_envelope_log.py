"""Pins for the oracle's IQ envelope, Hilbert envelope and log compression."""
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
FS, F0 = 40e6, 7e6
BW = 0.6 * F0


def test_fir_taps_symmetric_unit_dc_S227():
    h = oracle.fir_taps(65, BW / 2, FS)
    assert abs(h.sum() - 1.0) < 1e-14                     # DC gain 1 (reading #16)
    assert np.array_equal(h, h[::-1])                     # zero phase
    assert np.argmax(h) == 32


def test_fir_stopband_2f0():
    # mixing a tone at f0 leaves an image at 2 f0: the low-pass must reject it
    h = oracle.fir_taps(65, BW / 2, FS)
    j = np.arange(-32, 33)
    H = lambda f: abs(np.sum(h * np.exp(-2j * np.pi * f / FS * j)))
    assert 20 * math.log10(H(2 * F0)) < -40.0
    assert abs(H(0.0) - 1.0) < 1e-14


def test_zero_in_zero_out():
    assert np.all(oracle.iq_envelope(np.zeros((2, 512)), FS, F0, BW) == 0.0)
    assert np.all(oracle.hilbert_envelope(np.zeros(512)) == 0.0)


def test_tone_amplitude_S199():
    # A cos(2 pi f0 n / fs) -> envelope A away from the edges (2%);
    # the 65-tap filter gives much better (0.2%).
    A = 1.7
    n = np.arange(2048)
    x = A * np.cos(2 * np.pi * F0 * n / FS)
    env = oracle.iq_envelope(x, FS, F0, BW)
    assert np.max(np.abs(env[100:-100] - A)) <= 0.002 * A


def test_hilbert_integer_cycle_cosine_S208_corrected():
    # reading #27: S:208's f = 0.1 leaks; an integer number of cycles is exact
    n = np.arange(1024)
    x = np.cos(2 * np.pi * 0.125 * n)
    assert np.max(np.abs(oracle.hilbert_envelope(x) - 1.0)) < 1e-12


def test_impulse_peak_S209():
    x = np.zeros(512)
    x[200] = 1.0
    assert np.argmax(oracle.hilbert_envelope(x)) == 200
    assert np.argmax(oracle.iq_envelope(x, FS, F0, BW)) == 200


def test_scale_equivariance_and_sign_S221():
    rng = np.random.default_rng(0)
    x = rng.standard_normal(1024)
    e = oracle.iq_envelope(x, FS, F0, BW)
    assert np.max(np.abs(oracle.iq_envelope(3.0 * x, FS, F0, BW) - 3.0 * e)) <= 1e-12 * e.max()
    assert np.array_equal(oracle.iq_envelope(-x, FS, F0, BW), e)


def test_iq_vs_hilbert_gaussian_pulse_S223():
    # reading #27: pulse fbw 0.3 lies inside the 0.6 f0 band -> <= 5% rel L2
    n = np.arange(2048)
    sig_f = 0.3 * F0 / (2 * math.sqrt(2 * math.log(2)))
    sig = FS / (2 * math.pi * sig_f)
    x = np.exp(-(n - 1000.0) ** 2 / (2 * sig ** 2)) * np.cos(2 * np.pi * F0 * (n - 1000.0) / FS)
    e_iq = oracle.iq_envelope(x, FS, F0, BW)[64:-64]
    e_h = oracle.hilbert_envelope(x)[64:-64]
    assert np.linalg.norm(e_iq - e_h) / np.linalg.norm(e_h) <= 0.05
    # the envelope of a Gaussian-enveloped tone is the Gaussian itself
    g = np.exp(-(n - 1000.0) ** 2 / (2 * sig ** 2))[64:-64]
    assert np.linalg.norm(e_h - g) / np.linalg.norm(g) <= 0.01


def test_decimation_keeps_every_dth():
    rng = np.random.default_rng(1)
    x = rng.standard_normal(1000)
    e1 = oracle.iq_envelope(x, FS, F0, BW)
    e4 = oracle.iq_envelope(x, FS, F0, BW, decimation=4)
    assert len(e4) == 250 and np.array_equal(e4, e1[::4])


# ---------------------------------------------------------------- log
def test_log_endpoints_S257_S259():
    g = GOLD["log_endpoints"]
    DR = g["dr_db"]
    ref = 3.0
    x = np.array([ref, ref * 10 ** (-DR / 20), ref * 10 ** (-DR / 40), 0.0, ref * 1e-9])
    y, r = oracle.log_compress(x, DR, ref_mode=1, ref_value=ref)
    assert y[0] == g["at_ref"]
    assert abs(y[1] - g["at_minus_dr"]) < 1e-15
    assert abs(y[2] - g["at_minus_half_dr"]) < 1e-15
    assert y[3] == 0.0 and y[4] == 0.0
    u8 = oracle.to_u8(y)
    assert u8[0] == 255 and u8[1] == 0 and u8[2] == 128     # floor(127.5 + 0.5)


def test_log_monotone_bounded_S262():
    rng = np.random.default_rng(2)
    x = np.sort(rng.exponential(1.0, 10000))
    y, ref = oracle.log_compress(x, 50.0)
    assert ref == x.max()
    assert np.all(np.diff(y) >= 0) and y.min() >= 0 and y.max() == 1.0


def test_log_frame_max_scale_invariance_S263():
    rng = np.random.default_rng(3)
    x = rng.exponential(1.0, 5000)
    y1, _ = oracle.log_compress(x, 50.0)
    y2, _ = oracle.log_compress(x * 8.0, 50.0)     # power-of-two scale: exact in binary
    assert np.array_equal(y1, y2)


def test_log_all_zero_frame():
    y, ref = oracle.log_compress(np.zeros(100), 50.0)
    assert ref == 0.0 and np.all(y == 0.0)


# ------------------------------------------------- frequency compounding
# P:121 "frequency compounding through a bank of configurable bandpasses";
# S:186-189 (BandpassBank), S:213-218 (compound and its examples).
FS = 40e6
BAND_LO = (3.0e6, 2.0e6)      # 2 .. 4 MHz
BAND_HI = (8.0e6, 2.0e6)      # 7 .. 9 MHz (disjoint, equal widths)


def _tone(f, A, N=4096):
    n = np.arange(N)
    return A * np.cos(2 * np.pi * f * n / FS + 0.3)


def test_compound_single_band_weight_one_is_iq_demodulate():
    # single band, weight 1 -> identical to iq_demodulate
    x = np.random.default_rng(3).standard_normal(2048)
    e1 = oracle.compound(x, FS, ((7e6, 4.2e6, 1.0),))
    e2 = oracle.iq_envelope(x, FS, 7e6, 4.2e6)
    assert np.array_equal(e1, e2)


@pytest.mark.parametrize("wlo", [0.5, 0.3, 0.8])
def test_compound_tone_inside_one_band(wlo):
    # two disjoint bands, tone inside band 1 only -> w1 x single-band
    # envelope within 2% (band 2 rejects it below -40 dB); here the
    # single-band envelope of a tone of amplitude A is A, so the
    # closed form is w1 A.
    bands = ((*BAND_LO, wlo), (*BAND_HI, 1.0 - wlo))
    A = 1.7
    mid = slice(200, -200)
    e = oracle.compound(_tone(3.0e6, A), FS, bands)[mid]
    assert np.max(np.abs(e - wlo * A)) <= 0.02 * wlo * A
    e = oracle.compound(_tone(8.0e6, A), FS, bands)[mid]
    assert np.max(np.abs(e - (1 - wlo) * A)) <= 0.02 * (1 - wlo) * A


def test_compound_two_tones_one_per_band():
    # superposition across disjoint bands: w1 A1 + w2 A2 within 2%
    bands = ((*BAND_LO, 0.4), (*BAND_HI, 0.6))
    x = _tone(3.0e6, 2.0) + _tone(8.0e6, 0.5)
    e = oracle.compound(x, FS, bands)[200:-200]
    want = 0.4 * 2.0 + 0.6 * 0.5
    assert np.max(np.abs(e - want)) <= 0.02 * want


def test_compound_scale_equivariance_and_sign():
    # envelope(a x) = a envelope(x), envelope(-x) = envelope(x)
    bands = ((*BAND_LO, 0.5), (*BAND_HI, 0.5))
    x = np.random.default_rng(5).standard_normal(1024)
    e = oracle.compound(x, FS, bands)
    assert np.allclose(oracle.compound(3.5 * x, FS, bands), 3.5 * e, rtol=1e-12, atol=0)
    assert np.allclose(oracle.compound(-x, FS, bands), e, rtol=1e-12, atol=0)


def test_compound_reduces_speckle_variance():
    # uniform white-noise input -> the compounded envelope's variance
    # is <= the minimum single-band variance (speckle reduction), over >= 100
    # realisations.  With equal weights and disjoint equal-width bands the
    # band envelopes are independent, so the variance halves (bound: <= min).
    rng = np.random.default_rng(11)
    bands = ((*BAND_LO, 0.5), (*BAND_HI, 0.5))
    vc = vl = vh = 0.0
    R = 100
    for _ in range(R):
        x = rng.standard_normal(1024)
        vc += np.var(oracle.compound(x, FS, bands)[100:-100])
        vl += np.var(oracle.iq_envelope(x, FS, *BAND_LO)[100:-100])
        vh += np.var(oracle.iq_envelope(x, FS, *BAND_HI)[100:-100])
    assert vc / R <= min(vl, vh) / R
    assert vc / R <= 0.7 * min(vl, vh) / R      # and clearly so (~0.5)
