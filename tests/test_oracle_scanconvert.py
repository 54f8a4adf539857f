"""Pins for the oracle's scan conversion."""
import math

import numpy as np
import pytest

import oracle
from synth import configs


def sector(L=7, S=400, nx=41, nz=45, fov=60.0, dr_fs=40e6):
    o, d = configs.phased_lines(L, fov)
    ev = np.arange(L, dtype=np.int32)
    dr = configs.dr_mm(1540.0, dr_fs)
    sp = (S - 1) * dr / (nz - 1)
    return configs.Workload("sec", 16, 1, 0.22, 0.22, 3.5e6, L, S, L, 1, o, d, ev,
                            np.zeros((L, 3)), configs.SC_SECTOR_2D, (nx, 1, nz),
                            (-(nx - 1) / 2 * sp, 0.0, 0.0), (sp, sp, sp), fov_x_deg=fov,
                            fs_hz=dr_fs)


def pyramid(Lx=6, Ly=5, S=300, n=24, fovx=60.0, fovy=40.0):
    o, d = configs.phased_lines(Lx, fovx, Ly, fovy)
    L = Lx * Ly
    ev = np.arange(L, dtype=np.int32)
    sp = (S - 1) * configs.dr_mm() / (n - 1)
    return configs.Workload("pyr", 4, 4, 0.3, 0.3, 7e6, L, S, Lx, Ly, o, d, ev, np.zeros((L, 3)),
                            configs.SC_PYRAMID_3D, (n, n, n),
                            (-(n - 1) / 2 * sp, -(n - 1) / 2 * sp, 0.0), (sp, sp, sp),
                            fov_x_deg=fovx, fov_y_deg=fovy)


def small_linear():
    w = configs.c1()
    return w.replace(S=400, out_dims=(60, 1, 70), out_origin_mm=(-9.45, 0.0, 0.0),
                     out_spacing_mm=(0.32, 0.1, 0.11))


@pytest.mark.parametrize("mk", [small_linear, sector, pyramid])
def test_partition_of_unity_S309(mk):
    w = mk()
    y = np.full((w.L, w.S), 0.6180339887)
    img, mask = oracle.scan_convert(w, y)
    assert mask.sum() > 0
    assert np.max(np.abs(img[mask == 1] - 0.6180339887)) < 1e-12
    assert np.all(img[mask == 0] == 0.0)


@pytest.mark.parametrize("mk", [small_linear, sector, pyramid])
def test_monotone_bound_S315(mk):
    w = mk()
    rng = np.random.default_rng(5)
    y = rng.uniform(0.2, 0.9, (w.L, w.S))
    img, mask = oracle.scan_convert(w, y)
    v = img[mask == 1]
    assert v.min() >= y.min() - 1e-15 and v.max() <= y.max() + 1e-15


def test_grid_aligned_identity_S300():
    # line pitch = sample pitch = spacing = 2^-6 mm: every u, v is an exact
    # integer and the table is a pure index copy.
    s = 2.0 ** -6
    fs = 1000.0 * 1540.0 / (2.0 * s)        # dr = 2^-6 mm
    L, S = 9, 40
    xs = np.arange(L) * s
    o, d = configs.linear_lines(xs)
    ev = np.arange(L, dtype=np.int32)
    w = configs.Workload("id", L, 1, s, s, 7e6, L, S, L, 1, o, d, ev, np.zeros((L, 3)),
                         configs.SC_LINEAR_2D, (L, 1, S), (0.0, 0.0, 0.0), (s, s, s), fs_hz=fs)
    rng = np.random.default_rng(6)
    y = rng.uniform(0, 1, (L, S))
    img, mask = oracle.scan_convert(w, y)
    assert np.all(mask == 1)
    assert np.array_equal(img[:, 0, :], y.T)
    valid, idx, frac = oracle.sc_table(w)
    assert np.all(np.isin(frac[:, [0, 2]], (0.0, 1.0)))


@pytest.mark.parametrize("L,expect_i0,expect_f", [(7, 3, 0.0), (8, 3, 0.5)])
def test_sector_central_axis_symmetry_S301(L, expect_i0, expect_f):
    w = sector(L=L, nx=41)
    valid, idx, frac = oracle.sc_table(w)
    nx, nz = 41, 45
    centre = np.arange(nz) * nx + 20              # X = 0 column
    ok = valid[centre] == 1
    assert ok.sum() >= nz - 1
    assert np.all(idx[centre[ok], 0] == expect_i0)
    assert np.all(frac[centre[ok], 0] == expect_f)
    # mirror symmetry of validity about X = 0
    V = valid.reshape(nz, nx)
    assert np.array_equal(V, V[:, ::-1])


def test_linear_functions_reproduced_linear():
    # bilinear interpolation reproduces y = a*l + c*k + d exactly, so the
    # image equals a*u + c*v + d with u = (X - x0)/pitch, v = Z/dr (geometry)
    w = small_linear()
    a, c, d = 0.01, 0.002, 0.1
    l, k = np.meshgrid(np.arange(w.L), np.arange(w.S), indexing="ij")
    img, mask = oracle.scan_convert(w, a * l + c * k + d)
    X = w.out_origin_mm[0] + np.arange(w.out_dims[0]) * w.out_spacing_mm[0]
    Z = np.arange(w.out_dims[2]) * w.out_spacing_mm[2]
    ZZ, XX = np.meshgrid(Z, X, indexing="ij")
    expect = a * (XX + 9.45) / 0.3 + c * ZZ / configs.dr_mm() + d
    m = mask[:, 0, :] == 1
    assert np.max(np.abs(img[:, 0, :][m] - expect[m])) < 1e-10


def test_linear_functions_reproduced_sector():
    w = sector(L=9, nx=51, nz=47)
    k = np.arange(w.S)[None, :].repeat(w.L, 0)
    l = np.arange(w.L)[:, None].repeat(w.S, 1)
    sp = w.out_spacing_mm[0]
    X = w.out_origin_mm[0] + np.arange(51) * sp
    Z = np.arange(47) * sp
    ZZ, XX = np.meshgrid(Z, X, indexing="ij")
    img, mask = oracle.scan_convert(w, 0.001 * k.astype(float))
    m = mask[:, 0, :] == 1
    r_samples = np.hypot(XX, ZZ) / configs.dr_mm()
    assert np.max(np.abs(img[:, 0, :][m] - 0.001 * r_samples[m])) < 1e-11
    img, mask = oracle.scan_convert(w, 0.05 * l.astype(float))
    dth = math.radians(60.0) / 8
    u = np.arctan2(XX, ZZ) / dth + 4.0
    assert np.max(np.abs(img[:, 0, :][m] - 0.05 * u[m])) < 1e-11


def test_linear_functions_reproduced_pyramid():
    w = pyramid()
    k = np.broadcast_to(np.arange(w.S)[None, :], (w.L, w.S)).astype(float)
    img, mask = oracle.scan_convert(w, 0.001 * k)
    n = w.out_dims[0]
    sp = w.out_spacing_mm[0]
    X = w.out_origin_mm[0] + np.arange(n) * sp
    Y = w.out_origin_mm[1] + np.arange(n) * sp
    Z = np.arange(n) * sp
    ZZ, YY, XX = np.meshgrid(Z, Y, X, indexing="ij")
    r = np.sqrt(XX ** 2 + YY ** 2 + ZZ ** 2) / configs.dr_mm()
    m = mask == 1
    assert m.sum() > 100
    assert np.max(np.abs(img[m] - 0.001 * r[m])) < 1e-11


def _sector_valid_geometric(w):
    """Independent validity: inside the fan (|angle| <= fov/2) and within
    the imaged depth ((S-1) dr), from the pixel's polar coordinates."""
    nx, _, nz = w.out_dims
    sp = w.out_spacing_mm[0]
    X = w.out_origin_mm[0] + np.arange(nx) * sp
    Z = np.arange(nz) * sp
    ZZ, XX = np.meshgrid(Z, X, indexing="ij")
    half = math.radians(w.fov_x_deg / 2)
    inside = (np.abs(XX) <= ZZ * math.tan(half)) & (np.hypot(XX, ZZ) <= (w.S - 1) * configs.dr_mm())
    return inside


def test_sector_valid_count_C3():
    w = configs.c3()
    valid, idx, frac = oracle.sc_table(w)
    geo = _sector_valid_geometric(w)
    assert int(valid.sum()) == int(geo.sum())
    assert np.array_equal(valid.reshape(512, 512) == 1, geo)


def test_pyramid_valid_count_C4():
    w = configs.c4("b")
    valid, idx, frac = oracle.sc_table(w)
    n = 256
    sp = w.out_spacing_mm[0]
    X = w.out_origin_mm[0] + np.arange(n) * sp
    ZZ, YY, XX = np.meshgrid(np.arange(n) * sp, X, X, indexing="ij")
    half = math.radians(30.0)
    # inside the pyramid: |theta_y| <= 30 deg in the (y,z) plane and the
    # elevation of x above that plane <= 30 deg; radius within the depth
    rho_yz = np.hypot(YY, ZZ)
    geo = ((np.abs(YY) <= ZZ * math.tan(half)) & (np.abs(XX) <= rho_yz * math.tan(half)) &
           (np.sqrt(XX ** 2 + YY ** 2 + ZZ ** 2) <= (w.S - 1) * configs.dr_mm()))
    geo &= ZZ > 0
    diff = int(np.sum(valid.reshape(n, n, n).astype(bool) != geo))
    assert diff <= 8, diff                     # exact-boundary ties only
    assert abs(int(valid.sum()) - int(geo.sum())) <= 8


@pytest.mark.parametrize("dec", [2, 3])
def test_decimated_line_image_depth_axis_S224(dec):
    # with decimation d the line image holds k = d q at depth d q dr, so a
    # line image y[q] = d q (the full-rate sample index) scan-converts to
    # Z / dr exactly (linear interpolation reproduces linear functions)
    w = small_linear().replace(decimation=dec)
    Sd = w.S // dec
    q = np.arange(Sd)[None, :].repeat(w.L, 0).astype(float)
    img, mask = oracle.scan_convert(w, dec * q)
    Z = np.arange(w.out_dims[2]) * w.out_spacing_mm[2]
    expect = (Z / configs.dr_mm())[:, None].repeat(w.out_dims[0], 1)
    m = mask[:, 0, :] == 1
    assert m.any()
    assert np.max(np.abs(img[:, 0, :][m] - expect[m])) < 1e-9
    # the valid depth range ends at the last decimated sample (S:224 floor)
    zmax = (Sd - 1) * dec * configs.dr_mm()
    rows = np.where(m.any(1))[0]
    assert Z[rows].max() <= zmax + 1e-12 and Z[rows.max() + 1] > zmax if rows.max() + 1 < len(Z) else True


def test_pyramid_angular_axes_pinned_by_forward_steering_model():
    # Trilinear interpolation reproduces y = a lx + b ly + c k + d, so the
    # image must equal a u_x + b u_y + c v + d, where (u_x, u_y, v) come from
    # inverting the FORWARD steering model of reading #13, written here
    # independently of the oracle's atan2 form: a voxel P = r d(tx, ty) with
    # d = (sin tx, cos tx sin ty, cos tx cos ty) has r = |P|, tx = asin(X / r),
    # ty = atan(Y / Z); u = angle / dtheta + (L - 1)/2 (reading #14).
    # Lx != Ly and fov_x != fov_y, so a transposed line index or swapped
    # (fx, fy) fractions change the result.
    w = pyramid()                                  # Lx = 6, Ly = 5, 60 x 40 deg
    Lx, Ly, S = w.num_lines_x, w.num_lines_y, w.S
    a, b, c, d = 0.37, -0.61, 0.002, 0.25
    ly, lx, k = np.meshgrid(np.arange(Ly), np.arange(Lx), np.arange(S), indexing="ij")
    y = (a * lx + b * ly + c * k + d).reshape(Lx * Ly, S)   # line l = ly Lx + lx
    img, mask = oracle.scan_convert(w, y)
    n = w.out_dims[0]
    sp = w.out_spacing_mm[0]
    X = w.out_origin_mm[0] + np.arange(n) * sp
    Y = w.out_origin_mm[1] + np.arange(n) * sp
    Z = np.arange(n) * sp
    ZZ, YY, XX = np.meshgrid(Z, Y, X, indexing="ij")
    m = (mask == 1).reshape(n, n, n)
    assert m.sum() > 100
    r = np.sqrt(XX ** 2 + YY ** 2 + ZZ ** 2)
    tx = np.arcsin(XX[m] / r[m])
    ty = np.arctan(YY[m] / ZZ[m])
    ux = tx / (math.radians(60.0) / (Lx - 1)) + (Lx - 1) / 2
    uy = ty / (math.radians(40.0) / (Ly - 1)) + (Ly - 1) / 2
    v = r[m] / configs.dr_mm()
    expect = a * ux + b * uy + c * v + d
    got = img.reshape(n, n, n)[m]
    assert np.max(np.abs(got - expect)) < 1e-9
    # the angular axes separately (each must be reproduced on its own)
    img_x, _ = oracle.scan_convert(w, (1.0 * lx + 0 * k).reshape(Lx * Ly, S).astype(float))
    img_y, _ = oracle.scan_convert(w, (1.0 * ly + 0 * k).reshape(Lx * Ly, S).astype(float))
    assert np.max(np.abs(img_x.reshape(n, n, n)[m] - ux)) < 1e-9
    assert np.max(np.abs(img_y.reshape(n, n, n)[m] - uy)) < 1e-9
