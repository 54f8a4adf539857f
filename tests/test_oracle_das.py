"""Pins for the oracle's geometry and delay-and-sum (CPU, no GPU).

Each test pins oracle/oracle.c to something other than itself: values SPEC
prints (tests/golden/spec_examples.json), closed forms, invariants, special
cases, and a brute force on tiny inputs (SPEC acceptance #1).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth
from synth import configs

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def tiny_linear(n_el=16, pitch=0.3, S=256, **kw):
    xs = configs.element_x(n_el, pitch)
    o, d = configs.linear_lines(xs)
    ev = np.arange(n_el, dtype=np.int32)
    w = configs.Workload("tiny", n_el, 1, pitch, pitch, 7e6, n_el, S, n_el, 1, o, d, ev,
                         configs.tx_origins(o, ev, n_el), configs.SC_LINEAR_2D, (8, 1, 8),
                         (0, 0, 0), (0.1, 0.1, 0.1))
    return w.replace(**kw) if kw else w


# ------------------------------------------------------------ geometry
def test_linear_span_S56():
    g = GOLD["linear_span_mm"]
    pos = oracle.element_positions(g["elements"], 1, g["pitch_mm"], g["pitch_mm"])
    assert abs((pos[-1, 0] - pos[0, 0]) - g["value"]) < 1e-12
    assert abs(pos[:, 0].mean()) < 1e-12 and np.all(pos[:, 1:] == 0)


def test_matrix_grid_centered():
    pos = oracle.element_positions(32, 32, 0.3, 0.3)
    # channel ch = j*Nx + i (reading #15): channel 33 is (i=1, j=1)
    assert abs(pos[33, 0] - (1 - 15.5) * 0.3) < 1e-12 and abs(pos[33, 1] - (1 - 15.5) * 0.3) < 1e-12
    assert abs(pos[:, 0].mean()) < 1e-12 and abs(pos[:, 1].mean()) < 1e-12


def test_angle_grid_S66_S68():
    th = configs.angle_grid_rad(3, GOLD["three_lines_deg"]["fov_deg"])
    assert np.allclose(np.degrees(th), GOLD["three_lines_deg"]["value"], atol=1e-12)
    th = configs.angle_grid_rad(32, 60.0)
    assert abs(np.degrees(th[-1]) - GOLD["phased_extreme_deg"]["value"]) < 1e-12
    assert abs(np.degrees(th[0]) + GOLD["phased_extreme_deg"]["value"]) < 1e-12


def test_multiline_map_S57_S147():
    g = GOLD["multiline_255"]
    ev = configs.interleaved_line_events(g["events"], g["M"])
    assert len(ev) == g["lines"]
    for line, event in g["map"]:
        assert ev[line] == event


# ------------------------------------------------------------ delays
def test_delay_pythagoras_S78():
    g = GOLD["pythagoras_mm"]
    fs, c = 40e6, 1540.0
    # element 3 mm lateral of an on-axis focus at 20 mm: tau*(c/fs) = z + r
    tau = oracle.delay_samples([0, 0, 0], [0, 0, 1], [g["lateral_mm"], 0, 0], g["focus_mm"], fs, c)
    r = tau / fs * c * 1000.0 - g["focus_mm"]
    assert round(r, g["decimals"]) == g["value"]
    assert abs(r - math.sqrt(20.0 ** 2 + 3.0 ** 2)) < 1e-11


def test_round_trip_S432():
    g = GOLD["round_trip_us"]
    fs, c = 40e6, g["c_mps"]
    tau = oracle.delay_samples([0, 0, 0], [0, 0, 1], [0, 0, 0], g["depth_mm"], fs, c)
    assert round(tau / fs * 1e6, g["decimals"]) == g["value"]
    assert abs(tau - 2 * 0.020 / 1540.0 * 40e6) < 1e-9          # sample 1038.96


def test_steered_delay_law_of_cosines():
    # phased line at 25 deg, element at x=-2 mm: r^2 = z^2 + e^2 - 2 z e sin(25deg)*(-1)...
    th = math.radians(25.0)
    d = [math.sin(th), 0.0, math.cos(th)]
    ex, z, fs, c = -2.0, 17.0, 40e6, 1540.0
    tau = oracle.delay_samples([0, 0, 0], d, [ex, 0, 0], z, fs, c)
    r = math.sqrt(z * z + ex * ex - 2 * z * ex * math.sin(th))   # law of cosines, angle 90-th
    assert abs(tau - (z + r) / 1000.0 * fs / c) < 1e-9


def test_dr():
    assert abs(oracle.dr_mm(1540.0, 40e6) - 0.01925) < 1e-15


# ------------------------------------------------------------ DAS pins
def test_zero_in_zero_out_S136():
    w = tiny_linear()
    raw = np.zeros((w.num_events, w.C, w.S), np.int16)
    assert np.all(oracle.das(w, raw) == 0.0)


def _n_members_linear(n_el, pitch, l, k, F, dr):
    """Aperture count for a line at element centre l: elements whose lateral
    distance |e-l|*pitch is <= z/(2F), counted by integer offsets."""
    z = k * dr
    m = int(math.floor(z / (2 * F) / pitch + 1e-12))
    lo, hi = max(0, l - m), min(n_el - 1, l + m)
    return hi - lo + 1


@pytest.mark.parametrize("window", [configs.WIN_RECT, configs.WIN_HANN])
def test_impulse_on_line_channel_S137(window):
    # Channel l lies on line l (rho = 0): tau = k exactly, w(0) = 1, so an
    # impulse at sample n gives RF[l][k] = delta_kn / N(n).
    w = tiny_linear(n_el=16, S=256, window=window)
    l, n = 7, 150
    raw = np.zeros((w.num_events, w.C, w.S), np.int16)
    raw[l, l, n] = 1000
    rf = oracle.das(w, raw)
    dr = oracle.dr_mm(w.c_mps, w.fs_hz)
    N = _n_members_linear(16, 0.3, l, n, 1.0, dr)
    assert abs(rf[l, n] - 1000.0 / N) < 1e-9
    rf[l, n] = 0.0
    assert np.all(rf[l] == 0.0)


def test_constant_input_rect_returns_count_and_unity():
    # x == 1 everywhere, rect window: v = 1 for every member with tau <= S-1,
    # so RF = N (normalize none) and RF = 1 (count) -- the aperture count of S:153.
    n_el, S = 16, 256
    w = tiny_linear(n_el=n_el, S=S, window=configs.WIN_RECT, normalize=configs.NORM_NONE)
    raw = np.ones((w.num_events, w.C, w.S), np.int16)
    rf = oracle.das(w, raw)
    dr = oracle.dr_mm(w.c_mps, w.fs_hz)
    for l in (0, 5, 15):
        for k in range(0, 220, 7):
            assert abs(rf[l, k] - _n_members_linear(n_el, 0.3, l, k, 1.0, dr)) < 1e-12
    rf1 = oracle.das(w.replace(normalize=configs.NORM_COUNT), raw)
    assert np.all(np.abs(rf1[:, 1:220] - 1.0) < 1e-12)


def test_constant_input_hann_returns_weight_sum_north_star():
    # north_star: "a constant-channel input ... must return the apodization
    # weight sum": RF(normalize none) = sum_e 0.5 (1 + cos(pi rho_e / R)).
    n_el, S = 16, 256
    w = tiny_linear(n_el=n_el, S=S, window=configs.WIN_HANN, normalize=configs.NORM_NONE)
    raw = np.ones((w.num_events, w.C, w.S), np.int16)
    rf = oracle.das(w, raw)
    dr = oracle.dr_mm(w.c_mps, w.fs_hz)
    xs = configs.element_x(n_el, 0.3)
    for l in (2, 8):
        for k in range(1, 220, 11):
            R = k * dr / 2.0
            rho = np.abs(xs - xs[l])
            mem = 2.0 * rho <= k * dr
            expect = np.sum(0.5 * (1 + np.cos(np.pi * rho[mem] / R)))
            assert abs(rf[l, k] - expect) < 1e-12


def test_aperture_rule_S153():
    # Data only on channel 0; line 15 is 4.5 mm away: channel 0 joins the
    # aperture at z = 2 F rho = 9 mm (k = 467.5 -> 468), S = 400 never reaches it.
    w = tiny_linear(n_el=16, S=400)
    raw = np.zeros((w.num_events, w.C, w.S), np.int16)
    raw[:, 0, :] = 1234
    rf = oracle.das(w, raw)
    assert np.all(rf[15] == 0.0)
    # line 3 is 0.9 mm away: member from z = 1.8 mm (k >= 93.5 -> 94)
    k_in = int(math.ceil(2 * 0.9 / oracle.dr_mm(w.c_mps, w.fs_hz)))
    S_ok = 380  # beyond, tau > S-1 and zero padding (reading #10) applies
    assert np.all(rf[3, :k_in] == 0.0) and np.all(rf[3, k_in + 1:S_ok] != 0.0)


def test_linearity_S151():
    w = tiny_linear(n_el=16, S=256)
    rng = np.random.default_rng(1)
    X = rng.integers(-1000, 1000, (w.num_events, w.C, w.S)).astype(np.int16)
    Y = rng.integers(-1000, 1000, (w.num_events, w.C, w.S)).astype(np.int16)
    Z = (2 * X.astype(np.int32) - 3 * Y.astype(np.int32)).astype(np.int16)
    a, b, c = oracle.das(w, X), oracle.das(w, Y), oracle.das(w, Z)
    assert np.max(np.abs(c - (2 * a - 3 * b))) <= 1e-12 * np.max(np.abs(c))


def test_point_focus_C1_S447():
    w = configs.c1()
    raw = synth.channel_data_cpu(w)
    rf, env, y, ref = oracle.bmode_frame(w, raw)
    assert np.unravel_index(np.argmax(env), env.shape) == (32, 600)
    assert y.max() == 1.0


def test_translation_equivariance_S152():
    w = configs.c1()
    dr = configs.dr_mm()
    peaks = []
    for l in (20, 21):
        scat = np.array([[configs.element_x(64, 0.3)[l], 0.0, 400 * dr, 1.0]])
        raw = synth.channel_data_cpu(w, scat=scat)
        rf = oracle.das(w, raw, lines=np.arange(10, 32))
        env = oracle.iq_envelope(rf, w.fs_hz, 7e6, 4.2e6)
        peaks.append(np.unravel_index(np.argmax(env), env.shape))
    assert peaks[1][0] - peaks[0][0] == 1 and peaks[1][1] == peaks[0][1] == 400


def _brute_force_das(w, raw):
    """Independent NumPy brute force (SPEC acceptance #1): per line,
    per depth sample, vectorised over channels."""
    pos = np.stack(np.meshgrid((np.arange(w.elements_x) - (w.elements_x - 1) / 2) * w.pitch_x_mm,
                               (np.arange(w.elements_y) - (w.elements_y - 1) / 2) * w.pitch_y_mm,
                               indexing="xy"), -1).reshape(-1, 2)
    pos = np.concatenate([pos, np.zeros((len(pos), 1))], 1)
    dr = w.c_mps * 1e3 / (2 * w.fs_hz)
    out = np.zeros((w.L, w.S))
    allpos = pos
    for l in range(w.L):
        o, d = w.line_origin_mm[l], w.line_direction[l]
        x = raw[w.line_event[l]].astype(np.float64)
        if w.channel_element is not None:      # receive channel map
            els = np.asarray(w.channel_element[w.line_event[l]])
            x = x[els >= 0]
            pos = allpos[els[els >= 0]]
        else:
            pos = allpos
        xp = np.concatenate([x, np.zeros((x.shape[0], 2))], 1)
        rho = np.hypot(pos[:, 0] - o[0], pos[:, 1] - o[1])
        for k in range(w.S):
            z = k * dr
            mem = 2 * w.f_number * rho <= z
            if not mem.any():
                continue
            p = o + z * d
            r = np.linalg.norm(p[None, :] - pos, axis=1)
            tau = (z + r) * 1e-3 * w.fs_hz / w.c_mps
            i0 = np.floor(tau).astype(int)
            f = tau - i0
            ch = np.arange(len(pos))
            a = np.where((i0 >= 0) & (i0 < w.S), xp[ch, np.clip(i0, 0, w.S + 1)], 0.0)
            b = np.where((i0 + 1 >= 0) & (i0 + 1 < w.S), xp[ch, np.clip(i0 + 1, 0, w.S + 1)], 0.0)
            v = (1 - f) * a + f * b
            if getattr(w, "interpolation", 0) == 1:       # nearest (reading #32)
                i1 = np.floor(tau + 0.5).astype(int)
                v = np.where((i1 >= 0) & (i1 < w.S), xp[ch, np.clip(i1, 0, w.S + 1)], 0.0)
            u = rho / (z / (2 * w.f_number)) if z > 0 else np.zeros_like(rho)
            wt = 0.5 * (1 + np.cos(np.pi * u))
            out[l, k] = np.sum((wt * v)[mem]) / mem.sum()
    return out


@pytest.mark.parametrize("kind", ["linear", "phased", "matrix"])
def test_bruteforce_tiny_S570(kind):
    rng = np.random.default_rng({"linear": 2, "phased": 3, "matrix": 4}[kind])
    if kind == "linear":
        w = tiny_linear(n_el=16, S=256)
        ev = rng.integers(0, 8, w.L).astype(np.int32)
        w = w.replace(num_events=8, line_event=ev, tx_origin_mm=np.zeros((8, 3)))
    elif kind == "phased":
        o, d = configs.phased_lines(12, 50.0)
        ev = (np.arange(12) % 8).astype(np.int32)
        w = configs.Workload("tp", 16, 1, 0.22, 0.22, 3.5e6, 8, 256, 12, 1, o, d, ev,
                             np.zeros((8, 3)), configs.SC_SECTOR_2D, (8, 1, 8), (0, 0, 0),
                             (0.1, 0.1, 0.1), fov_x_deg=50.0)
    else:
        o, d = configs.phased_lines(4, 40.0, 3, 30.0)
        ev = (np.arange(12) % 8).astype(np.int32)
        w = configs.Workload("tm", 4, 4, 0.3, 0.3, 7e6, 8, 256, 4, 3, o, d, ev,
                             np.zeros((8, 3)), configs.SC_PYRAMID_3D, (8, 8, 8), (0, 0, 0),
                             (0.1, 0.1, 0.1), fov_x_deg=40.0, fov_y_deg=30.0)
    raw = rng.integers(-3000, 3000, (w.num_events, w.C, w.S)).astype(np.int16)
    a = oracle.das(w, raw)
    b = _brute_force_das(w, raw)
    assert np.max(np.abs(a - b)) <= 1e-9 * np.max(np.abs(b))


def test_determinism_threads():
    w = configs.c1()
    raw = synth.channel_data_cpu(w)
    a = oracle.das(w, raw, nthreads=1)
    b = oracle.das(w, raw, nthreads=7)
    assert np.array_equal(a, b)


# --------------------------------------- receive channel map (Table 1, f2)
# P:161 "only 64 channels usable" for the 128-element probe; S:102 active
# aperture; S:57/S:147 interleaved multi-line; P:337 Table-1 shapes.

@pytest.mark.parametrize("E,M,L", [(64, 1, 64), (64, 2, 127), (128, 1, 128), (128, 2, 255)])
def test_table1_shapes_P337(E, M, L):
    w = configs.table1(E, M)
    assert w.L == L and w.num_events == E and w.C == 64 and w.S * configs.dr_mm() >= 45.0
    assert w.line_event[-1] == E - 1
    if M == 2:
        assert w.line_event[L - 1] == E - 1 and w.line_event[3] == 1
    # every event records 64 contiguous elements holding its transmit position
    ex = configs.element_x(128, 0.3)
    for e in range(E):
        els = w.channel_element[e]
        assert np.array_equal(els, np.arange(els[0], els[0] + 64))
        assert ex[els[0]] - 0.15 <= w.tx_origin_mm[e, 0] <= ex[els[-1]] + 0.15


def test_identity_channel_map_equals_no_map():
    w = tiny_linear(n_el=16, S=256)
    rng = np.random.default_rng(8)
    raw = rng.integers(-3000, 3000, (w.num_events, w.C, w.S)).astype(np.int16)
    ident = np.tile(np.arange(16, dtype=np.int32), (w.num_events, 1))
    assert np.array_equal(oracle.das(w, raw), oracle.das(w.replace(channel_element=ident), raw))


def test_walking_aperture_constant_input_counts_recorded_members():
    # rect window, normalize none, x == 1: RF = number of RECORDED aperture
    # members wherever every member's tau <= S - 1 (the north-star pin,
    # restricted to the event's active channels)
    w0 = tiny_linear(n_el=32, S=512, window=configs.WIN_RECT, normalize=configs.NORM_NONE)
    chm = configs.walking_aperture(32, 8, 0.3, w0.tx_origin_mm[:, 0])
    w = w0.replace(channel_element=chm)
    raw = np.ones((w.num_events, 8, w.S), np.int16)
    rf = oracle.das(w, raw)
    ex = configs.element_x(32, 0.3)
    dr = configs.dr_mm()
    for l in (0, 9, 31):
        rec = ex[chm[w.line_event[l]]]
        for k in (40, 120, 200):
            n = int(np.sum(2.0 * w.f_number * np.abs(rec - w.line_origin_mm[l, 0]) <= k * dr))
            assert rf[l, k] == n


def test_bruteforce_walking_aperture_multiline_S570():
    w0 = tiny_linear(n_el=24, S=256)
    E, M = 12, 2
    ev = configs.interleaved_line_events(E, M)
    L = len(ev)
    o, d = configs.linear_lines(-(23 / 2) * 0.3 + np.arange(L) * (23 * 0.3 / (L - 1)))
    tx = configs.tx_origins(o, ev, E)
    chm = configs.walking_aperture(24, 10, 0.3, tx[:, 0])
    chm[3, 4] = -1                                   # an unused channel
    w = w0.replace(num_events=E, num_lines_x=L, line_origin_mm=o, line_direction=d, line_event=ev,
                   tx_origin_mm=tx, channel_element=chm)
    raw = np.random.default_rng(9).integers(-3000, 3000, (E, 10, w.S)).astype(np.int16)
    a = oracle.das(w, raw)
    b = _brute_force_das(w, raw)
    assert np.max(np.abs(a - b)) <= 1e-9 * np.max(np.abs(b))



@pytest.mark.parametrize("kind", ["linear", "phased"])
def test_bruteforce_nearest_interpolation_S125(kind):
    rng = np.random.default_rng(21)
    if kind == "linear":
        w = tiny_linear(n_el=16, S=256, interpolation=1)
    else:
        o, d = configs.phased_lines(12, 50.0)
        ev = (np.arange(12) % 8).astype(np.int32)
        w = configs.Workload("tp", 16, 1, 0.22, 0.22, 3.5e6, 8, 256, 12, 1, o, d, ev,
                             np.zeros((8, 3)), configs.SC_SECTOR_2D, (8, 1, 8), (0, 0, 0),
                             (0.1, 0.1, 0.1), fov_x_deg=50.0, interpolation=1)
    raw = rng.integers(-3000, 3000, (w.num_events, w.C, w.S)).astype(np.int16)
    a = oracle.das(w, raw)
    b = _brute_force_das(w, raw)
    assert np.max(np.abs(a - b)) <= 1e-9 * np.max(np.abs(b))
    # and it is not the linear result
    assert np.max(np.abs(a - oracle.das(w.replace(interpolation=0), raw))) > 1e-3 * np.max(np.abs(b))


def test_nearest_picks_rounded_sample_single_element():
    # one element, one line through it: tau(k) = k + |q|... here q = 0, so
    # tau = k exactly and both lookups return x[k]; with t0 = 0.4 samples the
    # nearest lookup still returns x[k] (k + 0.4 rounds down) and with t0 =
    # 0.6 it returns x[k + 1] (ties and above round up)
    w = tiny_linear(n_el=1, S=64, window=configs.WIN_RECT, normalize=configs.NORM_NONE, interpolation=1)
    w = w.replace(num_lines_x=1, line_origin_mm=np.zeros((1, 3)), line_direction=np.array([[0, 0, 1.0]]),
                  line_event=np.zeros(1, np.int32), num_events=1, tx_origin_mm=np.zeros((1, 3)))
    x = np.arange(64, dtype=np.int16)[None, None, :] * 3
    fs = w.fs_hz
    rf4 = oracle.das(w.replace(t0_s=0.4 / fs), x)[0]
    rf6 = oracle.das(w.replace(t0_s=0.6 / fs), x)[0]
    k = np.arange(10, 60)
    assert np.array_equal(rf4[k], 3.0 * k)
    assert np.array_equal(rf6[k], 3.0 * (k + 1))


def test_paper_3d_shape_P228_P337():
    # P:228 "512 (32 x 16) scanlines over a field of view of 60 deg", 70 mm
    # depth; P:347 384 channels; P:337 0.175 mm isotropic output
    w = configs.c4p()
    assert w.L == 512 and (w.num_lines_x, w.num_lines_y) == (32, 16)
    assert w.C == 384 and (w.S - 1) * configs.dr_mm() >= 70.0
    assert np.all(np.diff(np.sort(w.channel_element[0])) > 0)            # distinct elements
    th = np.degrees(np.arctan2(w.line_direction[:, 0],
                               np.hypot(w.line_direction[:, 1], w.line_direction[:, 2])))
    assert abs(th.max() - 30.0) < 1e-9 and abs(th.min() + 30.0) < 1e-9   # S:66 endpoints
    assert w.out_spacing_mm == (0.175, 0.175, 0.175)


# Window shape pinned by its textbook landmarks (S:125 lists {rectangular,
# hann, hamming}; reading #9 maps the aperture edge rho = R to u = 1):
# Hann is 0 at the edge, 1/2 half way, 1 on the axis; Hamming is 0.08 at the
# edge (0.54 - 0.46), 0.54 half way and 1 on the axis; rect is 1 throughout.
@pytest.mark.parametrize("window,edge,half,axis", [
    (configs.WIN_HANN, 0.0, 0.5, 1.0),
    (configs.WIN_HAMMING, 0.08, 0.54, 1.0),
    (configs.WIN_RECT, 1.0, 1.0, 1.0),
])
def test_window_landmarks_single_element_S125(window, edge, half, axis):
    # binary-exact geometry: dr = 2^-6 mm (fs = 49.28 MHz at c = 1540 m/s),
    # pitch 2^-4 mm, F = 1.  The neighbour of line l sits at rho = 2^-4 mm:
    # it joins the aperture at k = 8 (2 F rho = 8 dr exactly, u = rho / R = 1)
    # and is half way in at k = 16 (u = 1/2).  Only one channel carries data
    # (constant 1000, every tau inside the record), normalize = none, so
    # RF[l][k] = 1000 w(u) isolates the window value of that one element.
    fs = 1000.0 * 1540.0 / (2.0 * 2.0 ** -6)
    w = tiny_linear(n_el=16, pitch=2.0 ** -4, S=64).replace(fs_hz=fs, window=window,
                                                            normalize=configs.NORM_NONE)
    assert oracle.dr_mm(w.c_mps, w.fs_hz) == 2.0 ** -6
    l = 7
    raw = np.zeros((w.num_events, w.C, w.S), np.int16)
    raw[l, l + 1, :] = 1000                       # the neighbour at rho = pitch
    rf = oracle.das(w, raw)
    assert np.all(rf[l, :8] == 0.0)               # not yet a member
    assert abs(rf[l, 8] - 1000.0 * edge) < 1e-9   # u = 1: the aperture edge
    assert abs(rf[l, 16] - 1000.0 * half) < 1e-9  # u = 1/2
    # the line's own element (rho = 0, u = 0 at every depth, reading #9)
    raw2 = np.zeros_like(raw)
    raw2[l, l, :] = 1000
    rf2 = oracle.das(w, raw2)
    assert np.all(np.abs(rf2[l, :40] - 1000.0 * axis) < 1e-9)
    # the weight is monotone in u (edge -> axis) along the entering element
    seg = rf[l, 8:40]
    assert np.all(np.diff(seg) >= -1e-9) if edge <= axis else True
