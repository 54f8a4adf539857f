"""Pins for the PSF/FWHM measurement (SPEC measure_psf examples)."""
import numpy as np

from psf import fwhm, measure_psf


def test_gaussian_blob_fwhm_S531():
    # sigma_lateral = 0.4 mm -> FWHM = 2 sqrt(2 ln 2) 0.4 = 0.9419 mm +- 1 sample spacing
    dx = 0.0225
    x = np.arange(-200, 201) * dx
    z = np.arange(0, 1200) * 0.019
    sig_x, sig_z, z0 = 0.4, 0.25, 12.0
    img = np.exp(-x[:, None] ** 2 / (2 * sig_x ** 2) - (z[None, :] - z0) ** 2 / (2 * sig_z ** 2))
    r = measure_psf(img, dx, 0.019, z0, lateral_origin=x[0])
    assert abs(r["lateral_fwhm"] - 2 * np.sqrt(2 * np.log(2)) * 0.4) <= dx
    assert abs(r["axial_fwhm"] - 2 * np.sqrt(2 * np.log(2)) * 0.25) <= 0.019
    assert abs(r["peak_depth"] - z0) <= 0.019 and abs(r["peak_lateral"]) <= dx


def test_symmetric_profile_same_both_directions_S532():
    p = np.exp(-np.linspace(-3, 3, 121) ** 2)
    assert abs(fwhm(p, 0.1) - fwhm(p[::-1], 0.1)) <= 1e-9


def test_peak_at_boundary_is_flagged():
    p = np.linspace(1.0, 0.0, 50)
    assert np.isnan(fwhm(p, 0.1))
