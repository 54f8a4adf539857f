"""GPU parity: the CUDA path (through the C ABI) vs the binary64 oracle on the
same seeded int16 input (T3/T4/T5).  Gates (north_star): RF normwise <= 1e-4,
<= 0.01 dB on the log-compressed line image and on the scan-converted image,
u8 within 1 LSB, scan-conversion integer indices bit-exact."""
import numpy as np
import pytest

import oracle
from synth import configs

from gpu_util import DB_TOL, RF_TOL, db_err, oracle_chain, raw_frames, rf_err, run_gpu

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1711_06127_b200 import SupraBF  # noqa: E402
from paper_1711_06127_b200 import binding as B  # noqa: E402


def check_frame(w, raw_np, rf_g, y_g, lines=None):
    """Oracle for one frame; if ``lines`` is given only those lines are
    compared (the frame max then comes from the GPU side's own maximum,
    compared separately via the envelope)."""
    rf_o, env_o = oracle_chain(w, raw_np, lines=lines)
    sel = slice(None) if lines is None else lines
    e_rf = rf_err(rf_g[sel], rf_o)
    if lines is None:
        y_o, ref = oracle.log_compress(env_o, w.dynamic_range_db, w.reference_mode, w.reference_value)
        e_db = db_err(y_g, y_o, w.dynamic_range_db)
    else:
        e_db = None
    return e_rf, e_db, rf_o, env_o


# ------------------------------------------------------------------ C1
def test_c1_point_target_full_chain():
    w = configs.c1()
    raw = raw_frames(w, 1)
    bf = SupraBF(w)
    rf_g, y_g = run_gpu(bf, raw, 1)
    e_rf, e_db, rf_o, env_o = check_frame(w, raw[0].cpu().numpy(), rf_g[0], y_g[0])
    assert e_rf <= RF_TOL, e_rf
    assert e_db <= DB_TOL, e_db
    assert np.unravel_index(np.argmax(y_g[0]), y_g[0].shape) == (32, 600)
    # scan conversion of the GPU line image vs the oracle chain's image
    y_o, _ = oracle.log_compress(env_o, 50.0)
    img_o, mask_o = oracle.scan_convert(w, y_o)
    li = torch.from_numpy(y_g).cuda()
    img = bf.empty_img(1)
    mask = bf.empty_mask()
    bf.scanconvert(li, 1, img, mask)
    torch.cuda.synchronize()
    assert np.array_equal(mask.cpu().numpy(), mask_o)
    assert db_err(img.cpu().numpy()[0], img_o) <= DB_TOL


@pytest.mark.parametrize("over", [
    dict(window=configs.WIN_RECT),
    dict(window=configs.WIN_HAMMING, normalize=configs.NORM_NONE),
    dict(f_number=1.7),
    dict(t0_s=-2.5e-7),
    dict(t0_s=3e-7, fir_taps=33),
    dict(reference_mode=configs.REF_FIXED, reference_value=5000.0),
    dict(interpolation=configs.INTERP_NEAREST),
    dict(interpolation=configs.INTERP_NEAREST, window=configs.WIN_HAMMING, t0_s=1e-7),
    dict(fir_taps=129),                       # longest FIR (P = 64)
    dict(fir_taps=1),                         # degenerate FIR: env = 2|RF| scaled by the one tap
    dict(f_number=0.02),                      # whole array from the first samples
    dict(f_number=6.0),                       # tiny aperture: N(k) = 0 for most shallow k
])
def test_c1_variants(over):
    w = configs.c1(**over)
    raw = raw_frames(w, 1)
    bf = SupraBF(w)
    rf_g, y_g = run_gpu(bf, raw, 1)
    rf_o, env_o = oracle_chain(w, raw[0].cpu().numpy())
    assert rf_err(rf_g[0], rf_o) <= RF_TOL
    y_o, _ = oracle.log_compress(env_o, w.dynamic_range_db, w.reference_mode, w.reference_value)
    assert db_err(y_g[0], y_o) <= DB_TOL


def test_c1_u8_outputs_within_one_lsb():
    w = configs.c1(line_output_type=configs.T_U8, sc_output_type=configs.T_U8)
    raw = raw_frames(w, 1)
    bf = SupraBF(w)
    _, y_g = run_gpu(bf, raw, 1, want_rf=False)
    _, env_o = oracle_chain(w, raw[0].cpu().numpy())
    y_o, _ = oracle.log_compress(env_o, 50.0)
    u8_o = oracle.to_u8(y_o)
    assert y_g.dtype == np.uint8
    assert np.max(np.abs(y_g[0].astype(int) - u8_o.astype(int))) <= 1


def test_zero_frame_and_noop():
    w = configs.c1()
    bf = SupraBF(w, max_frames=2)
    raw = torch.zeros((2, w.num_events, w.C, w.S), dtype=torch.int16, device="cuda")
    rf_g, y_g = run_gpu(bf, raw, 2)
    assert np.all(rf_g == 0) and np.all(y_g == 0)
    bf.beamform(raw, 0, line_img=bf.empty_line_img(1))   # frames = 0: no-op
    with pytest.raises(B.SupraError):
        bf.beamform(raw, 3, line_img=bf.empty_line_img(3))
    with pytest.raises(B.SupraError):
        bf.beamform(raw, 1)


def test_envelope_log_standalone_matches_fused():
    w = configs.c1()
    raw = raw_frames(w, 1)
    bf = SupraBF(w)
    rf = bf.empty_rf(1)
    li = bf.empty_line_img(1)
    bf.beamform(raw, 1, rf=rf, line_img=li)
    li2 = bf.empty_line_img(1)
    bf.envelope_log(rf, 1, li2)
    torch.cuda.synchronize()
    assert torch.equal(li, li2)


# ------------------------------------------------------------------ C2
def test_c2_batch_parity_and_batch_invariance():
    w = configs.c2()
    F = 6                                  # FB groups of 4 + a ragged 2
    raw = raw_frames(w, F)
    bf = SupraBF(w, max_frames=F)
    rf_g, y_g = run_gpu(bf, raw, F)
    for f in (0, 3, 5):
        e_rf, e_db, _, _ = check_frame(w, raw[f].cpu().numpy(), rf_g[f], y_g[f])
        assert e_rf <= RF_TOL, (f, e_rf)
        assert e_db <= DB_TOL, (f, e_db)
    # frames are independent: any multi-frame batch gives bitwise the same
    # result (one sum order per configuration; all shapes are covered in
    # test_parity_shapes_gpu.py) ...
    rf2, y2 = run_gpu(bf, raw[4:6], 2)
    assert np.array_equal(rf2[1], rf_g[5]) and np.array_equal(y2[1], y_g[5])
    # ... and a single frame (the warp-split kernel, its own sum order)
    # agrees to float32 rounding
    rf1, y1 = run_gpu(bf, raw[5:6], 1)
    assert rf_err(rf1[0], rf_g[5].astype(np.float64)) <= 1e-6
    assert db_err(y1[0], y_g[5].astype(np.float64)) <= 1e-4
    # determinism
    rf_b, y_b = run_gpu(bf, raw, F)
    assert np.array_equal(rf_b, rf_g) and np.array_equal(y_b, y_g)


def test_c2b_multiline_parity():
    w = configs.c2("b")
    raw = raw_frames(w, 1)
    bf = SupraBF(w)
    rf_g, y_g = run_gpu(bf, raw, 1)
    e_rf, e_db, _, _ = check_frame(w, raw[0].cpu().numpy(), rf_g[0], y_g[0])
    assert e_rf <= RF_TOL and e_db <= DB_TOL, (e_rf, e_db)


# ------------------------------------------------------------------ C3
def test_c3_sector_parity_and_indices():
    w = configs.c3()
    raw = raw_frames(w, 1)
    bf = SupraBF(w)
    rf_g, y_g = run_gpu(bf, raw, 1)
    e_rf, e_db, rf_o, env_o = check_frame(w, raw[0].cpu().numpy(), rf_g[0], y_g[0])
    assert e_rf <= RF_TOL, e_rf
    assert e_db <= DB_TOL, e_db
    valid_o, idx_o, _ = oracle.sc_table(w)
    valid_g, idx_g = bf.sc_indices()
    assert np.array_equal(valid_g, valid_o)
    m = valid_o == 1
    assert np.array_equal(idx_g[m], idx_o[m])
    y_o, _ = oracle.log_compress(env_o, 50.0)
    img_o, mask_o = oracle.scan_convert(w, y_o)
    img = bf.empty_img(1)
    mask = bf.empty_mask()
    bf.scanconvert(torch.from_numpy(y_g).cuda(), 1, img, mask)
    torch.cuda.synchronize()
    assert np.array_equal(mask.cpu().numpy(), mask_o)
    assert db_err(img.cpu().numpy()[0], img_o) <= DB_TOL


# ------------------------------------------------------------------ C4
@pytest.mark.parametrize("variant", ["a", "b"])
def test_c4_sampled_lines(variant):
    w = configs.c4(variant)
    raw = raw_frames(w, 1)
    bf = SupraBF(w)
    rf_g, y_g = run_gpu(bf, raw, 1)
    rng = np.random.default_rng(7)
    lines = np.sort(np.concatenate([[0, 2047, 2080, 4095],
                                    rng.choice(4096, 12, replace=False)])).astype(np.int32)
    e_rf, _, rf_o, env_o = check_frame(w, raw[0].cpu().numpy(), rf_g[0], None, lines=lines)
    assert e_rf <= RF_TOL, e_rf
    # envelope parity on the sampled lines, in dB against the oracle's scale
    # (the log of a ratio of envelopes only needs the envelopes to agree)
    li = bf.empty_line_img(1)
    rf_t = torch.from_numpy(rf_g).cuda()
    # fixed reference = the oracle's max over the sampled lines: y comparable line by line
    ref = float(env_o.max())
    bf2 = SupraBF(w.replace(reference_mode=configs.REF_FIXED, reference_value=ref))
    bf2.envelope_log(rf_t, 1, li)
    torch.cuda.synchronize()
    y_o, _ = oracle.log_compress(env_o, 50.0, ref_mode=1, ref_value=ref)
    assert db_err(li.cpu().numpy()[0][lines], y_o) <= DB_TOL


def test_c4_scan_conversion_indices_and_values():
    w = configs.c4("b")
    bf = SupraBF(w)
    valid_o, idx_o, _ = oracle.sc_table(w)
    valid_g, idx_g = bf.sc_indices()
    assert int(valid_o.sum()) == 5788032
    assert np.array_equal(valid_g, valid_o)
    m = valid_o == 1
    assert np.array_equal(idx_g[m], idx_o[m])
    # values on a seeded synthetic line image fed to both sides
    rng = np.random.default_rng(11)
    y = rng.uniform(0, 1, (w.L, w.S))
    img_o, mask_o = oracle.scan_convert(w, y)
    img = bf.empty_img(1)
    mask = bf.empty_mask()
    bf.scanconvert(torch.from_numpy(y.astype(np.float32))[None].cuda(), 1, img, mask)
    torch.cuda.synchronize()
    assert np.array_equal(mask.cpu().numpy(), mask_o)
    # y rounded to f32 at the input (<= 3e-8) + f32 blend: well inside 0.01 dB
    assert db_err(img.cpu().numpy()[0], img_o) <= DB_TOL


def test_c2_scan_conversion_indices():
    w = configs.c2()
    bf = SupraBF(w)
    valid_o, idx_o, _ = oracle.sc_table(w)
    valid_g, idx_g = bf.sc_indices()
    assert np.array_equal(valid_g, valid_o)
    m = valid_o == 1
    assert np.array_equal(idx_g[m][:, [0, 2]], idx_o[m][:, [0, 2]])


def test_c2_bench_launch_configuration():
    """Full size, exactly the launch bench.py times: 100 frames per call
    (das_fused<16,4> over 96 frames + a <4,8> remainder launch for 4), f32
    line image, u8 B-mode.
    Sampled frames vs the oracle chain: line image <= 0.01 dB, B-mode u8
    within 1 LSB of the oracle's u8 of its own scan conversion."""
    w = configs.c2(sc_output_type=configs.T_U8)
    F = 100
    raw = raw_frames(w, F)
    bf = SupraBF(w, max_frames=F)
    li = bf.empty_line_img(F)
    img = bf.empty_img(F)
    mask = bf.empty_mask()
    bf.beamform(raw, F, line_img=li)
    bf.scanconvert(li, F, img, mask)
    torch.cuda.synchronize()
    for f in (0, 57, 99):
        raw_np = raw[f].cpu().numpy()
        rf_o, env_o = oracle_chain(w, raw_np)
        y_o, _ = oracle.log_compress(env_o, 50.0)
        assert db_err(li[f].cpu().numpy(), y_o) <= DB_TOL
        img_o, mask_o = oracle.scan_convert(w, y_o)
        u8_o = oracle.to_u8(img_o)
        got = img[f].cpu().numpy()
        assert np.max(np.abs(got.astype(int) - u8_o.astype(int))) <= 1
        if f == 0:
            assert np.array_equal(mask.cpu().numpy(), mask_o)
    del raw


# ------------------------------------------------- scanline-block split (8e)
@pytest.mark.parametrize("out_type", [configs.T_F32, configs.T_U8])
def test_line_range_split_equals_fused_c2(out_type):
    """beamform_lines on two line blocks + max of the two block maxima +
    log_compress per block == the fused single call, bitwise (same kernels,
    same arithmetic; max is exact)."""
    w = configs.c2(line_output_type=out_type)
    F = 3
    raw = raw_frames(w, F)
    bf = SupraBF(w, max_frames=F)
    li = bf.empty_line_img(F)
    bf.beamform(raw, F, line_img=li)
    env = torch.empty((F, w.L, w.S), dtype=torch.float32, device="cuda")
    fm = [torch.empty(F, dtype=torch.float32, device="cuda") for _ in range(2)]
    blocks = [(0, 100), (100, w.L - 100)]
    for (a, n), m in zip(blocks, fm):
        bf.beamform_lines(raw, F, a, n, env, m)
    gmax = torch.maximum(fm[0], fm[1])
    li2 = bf.empty_line_img(F)
    for a, n in blocks:
        bf.log_compress(env, F, a, n, gmax, li2)
    torch.cuda.synchronize()
    assert torch.equal(li, li2)
    # the envelope itself vs the oracle on one frame (RF-level parity is covered above)
    _, env_o = oracle_chain(w, raw[1].cpu().numpy())
    e = env[1].cpu().numpy().astype(np.float64)
    assert np.max(np.abs(e - env_o)) / np.max(env_o) <= 1e-4
    with pytest.raises(B.SupraError):
        bf.beamform_lines(raw, F, 200, 100, env, gmax)       # range past L


def test_c4b_scanline_block_split_equals_fused():
    """Latency mode for one C4b volume: 4 event-aligned scanline blocks
    (what 4 ranks of dist.ShardedVolume run) reproduce the fused volume
    bitwise, u8 line image."""
    from paper_1711_06127_b200.dist import shard_lines
    w = configs.c4("b", line_output_type=configs.T_U8)
    raw = raw_frames(w, 1)
    bf = SupraBF(w)
    li = bf.empty_line_img(1)
    bf.beamform(raw, 1, line_img=li)
    env = torch.empty((1, w.L, w.S), dtype=torch.float32, device="cuda")
    G = 4
    blocks = [shard_lines(w.L, G, r, 4 * w.num_lines_x) for r in range(G)]
    fms = []
    for a, n in blocks:
        m = torch.empty(1, dtype=torch.float32, device="cuda")
        bf.beamform_lines(raw, 1, a, n, env, m)
        fms.append(m)
    gmax = torch.stack(fms).max(0).values
    li2 = bf.empty_line_img(1)
    for a, n in blocks:
        bf.log_compress(env, 1, a, n, gmax, li2)
    torch.cuda.synchronize()
    assert torch.equal(li, li2)


# ------------------------------------------------- frequency compounding
# P:121 "frequency compounding through a bank of configurable bandpasses";
# env = sum_b w_b env_b, fused into the DAS epilogue.
BANDS_2 = ((5.5e6, 2.4e6, 0.5), (8.5e6, 2.4e6, 0.5))
BANDS_3 = ((5.0e6, 2.0e6, 0.25), (7.0e6, 2.0e6, 0.5), (9.0e6, 2.0e6, 0.25))


def test_c1_frequency_compounding_full_chain():
    w = configs.c1(bands=BANDS_2)
    raw = raw_frames(w, 1)
    bf = SupraBF(w)
    rf_g, y_g = run_gpu(bf, raw, 1)
    rf_o, env_o = oracle_chain(w, raw[0].cpu().numpy())
    assert rf_err(rf_g[0], rf_o) <= RF_TOL
    y_o, _ = oracle.log_compress(env_o, w.dynamic_range_db)
    assert db_err(y_g[0], y_o) <= DB_TOL
    # the standalone epilogue gives bitwise the fused result
    li2 = bf.empty_line_img(1)
    bf.envelope_log(torch.from_numpy(rf_g).cuda(), 1, li2)
    torch.cuda.synchronize()
    assert np.array_equal(li2.cpu().numpy(), y_g)
    # and compounding is really applied: the single-band image differs
    _, y1 = run_gpu(SupraBF(configs.c1()), raw, 1, want_rf=False)
    assert db_err(y1[0], y_g[0].astype(np.float64)) > 0.1


def test_c2_frequency_compounding_batch():
    w = configs.c2(bands=BANDS_3)
    F = 3
    raw = raw_frames(w, F)
    bf = SupraBF(w, max_frames=F)
    rf_g, y_g = run_gpu(bf, raw, F)
    for f in (0, 2):
        e_rf, e_db, _, _ = check_frame(w, raw[f].cpu().numpy(), rf_g[f], y_g[f])
        assert e_rf <= RF_TOL, (f, e_rf)
        assert e_db <= DB_TOL, (f, e_db)


# ---------------------------------- Table-1 acquisition shapes (f2)
@pytest.mark.parametrize("E,M", [(64, 1), (128, 2)])
def test_table1_shape_full_chain(E, M):
    w = configs.table1(E, M)
    raw = raw_frames(w, 1)
    bf = SupraBF(w)
    rf_g, y_g = run_gpu(bf, raw, 1)
    e_rf, e_db, _, _ = check_frame(w, raw[0].cpu().numpy(), rf_g[0], y_g[0])
    assert e_rf <= RF_TOL, e_rf
    assert e_db <= DB_TOL, e_db


def test_table1_batch_and_scan_conversion():
    w = configs.table1(64, 2, sc_output_type=configs.T_U8)
    F = 3
    raw = raw_frames(w, F)
    bf = SupraBF(w, max_frames=F)
    rf_g, y_g = run_gpu(bf, raw, F)
    e_rf, e_db, _, _ = check_frame(w, raw[2].cpu().numpy(), rf_g[2], y_g[2])
    assert e_rf <= RF_TOL and e_db <= DB_TOL, (e_rf, e_db)
    valid_o, idx_o, _ = oracle.sc_table(w)
    valid_g, idx_g = bf.sc_indices()
    assert np.array_equal(valid_g, valid_o)
    assert np.array_equal(idx_g[valid_o.astype(bool)], idx_o[valid_o.astype(bool)])



def test_c2_nearest_interpolation_batch():
    w = configs.c2(interpolation=configs.INTERP_NEAREST)
    F = 2
    raw = raw_frames(w, F)
    bf = SupraBF(w, max_frames=F)
    rf_g, y_g = run_gpu(bf, raw, F)
    e_rf, e_db, _, _ = check_frame(w, raw[1].cpu().numpy(), rf_g[1], y_g[1])
    assert e_rf <= RF_TOL and e_db <= DB_TOL, (e_rf, e_db)


# ------------------------------ the paper's 3D shape (f4)
def test_c4p_paper_3d_sampled_lines_and_indices():
    w = configs.c4p()
    raw = raw_frames(w, 1)
    bf = SupraBF(w)
    rf_g, _ = run_gpu(bf, raw, 1)
    rng = np.random.default_rng(17)
    lines = np.sort(np.concatenate([[0, 255, 256, 511], rng.choice(512, 8, replace=False)])).astype(np.int32)
    e_rf, _, _, _ = check_frame(w, raw[0].cpu().numpy(), rf_g[0], None, lines=lines)
    assert e_rf <= RF_TOL, e_rf
    valid_o, idx_o, _ = oracle.sc_table(w)
    valid_g, idx_g = bf.sc_indices()
    assert np.array_equal(valid_g, valid_o)
    v = valid_o.astype(bool)
    assert np.array_equal(idx_g[v], idx_o[v])


# ----------------------------------------- envelope decimation (f4)
@pytest.mark.parametrize("dec", [2, 3])
def test_c1_decimation_full_chain(dec):
    w = configs.c1(decimation=dec)
    raw = raw_frames(w, 1)
    bf = SupraBF(w)
    rf_g, y_g = run_gpu(bf, raw, 1)
    assert y_g.shape == (1, w.L, w.S // dec)
    rf_o, env_o = oracle_chain(w, raw[0].cpu().numpy())
    assert rf_err(rf_g[0], rf_o) <= RF_TOL
    y_o, _ = oracle.log_compress(env_o, w.dynamic_range_db)
    assert db_err(y_g[0], y_o) <= DB_TOL
    # standalone epilogue: bitwise the fused result
    li2 = bf.empty_line_img(1)
    bf.envelope_log(torch.from_numpy(rf_g).cuda(), 1, li2)
    torch.cuda.synchronize()
    assert np.array_equal(li2.cpu().numpy(), y_g)
    # scan conversion of the decimated line image: bit-exact indices, values
    img, mask = bf.empty_img(1), bf.empty_mask()
    bf.scanconvert(torch.from_numpy(y_g).cuda(), 1, img, mask)
    torch.cuda.synchronize()
    img_o, mask_o = oracle.scan_convert(w, y_o)
    assert np.array_equal(mask.cpu().numpy(), mask_o)
    assert db_err(img.cpu().numpy()[0], img_o) <= DB_TOL
    valid_o, idx_o, _ = oracle.sc_table(w)
    valid_g, idx_g = bf.sc_indices()
    v = valid_o.astype(bool)
    assert np.array_equal(valid_g, valid_o) and np.array_equal(idx_g[v], idx_o[v])


def test_c2_decimation_batch():
    w = configs.c2(decimation=4, line_output_type=configs.T_U8)
    F = 3
    raw = raw_frames(w, F)
    bf = SupraBF(w, max_frames=F)
    rf_g, y_g = run_gpu(bf, raw, F)
    rf_o, env_o = oracle_chain(w, raw[1].cpu().numpy())
    assert rf_err(rf_g[1], rf_o) <= RF_TOL
    y_o, _ = oracle.log_compress(env_o, w.dynamic_range_db)
    assert np.max(np.abs(y_g[1].astype(int) - oracle.to_u8(y_o).astype(int))) <= 1


# ------------------------- FIR epilogue on 16-frame batches (<16,4>; 65 and 33 taps)
@pytest.mark.parametrize("over", [dict(), dict(reference_mode=configs.REF_FIXED, reference_value=800.0,
                                               line_output_type=configs.T_U8),
                                  dict(fir_taps=33)])            # 33 taps: shorter halos
def test_c2_sixteen_frame_batch_epilogue(over):
    w = configs.c2(**over)
    F = 16
    raw = raw_frames(w, F)
    bf = SupraBF(w, max_frames=F)
    rf_g, y_g = run_gpu(bf, raw, F)
    for f in (0, 5, 15):
        rf_o, env_o = oracle_chain(w, raw[f].cpu().numpy())
        assert rf_err(rf_g[f], rf_o) <= RF_TOL
        y_o, _ = oracle.log_compress(env_o, w.dynamic_range_db, w.reference_mode, w.reference_value)
        if w.line_output_type == configs.T_U8:
            assert np.max(np.abs(y_g[f].astype(int) - oracle.to_u8(y_o).astype(int))) <= 1
        else:
            assert db_err(y_g[f], y_o) <= DB_TOL, f


# ----------------------- one-call raw -> B-mode (log compression inside SC)
@pytest.mark.parametrize("name,F,over", [
    ("C2", 16, dict(sc_output_type=configs.T_U8)),          # linear, tiled SC, frame max
    ("C2", 3, dict()),                                      # f32 image
    ("C3", 2, dict(sc_output_type=configs.T_U8)),           # sector table SC
    ("C1", 1, dict(reference_mode=configs.REF_FIXED, reference_value=3000.0)),
    ("C1", 1, dict(decimation=2)),
])
def test_beamform_bmode_equals_two_calls(name, F, over):
    w = configs.CONFIGS[name](**over)
    raw = raw_frames(w, F)
    bf = SupraBF(w, max_frames=F)
    li = torch.empty((F, w.L, w.S // w.decimation), dtype=torch.float32, device="cuda")
    bf2 = SupraBF(w.replace(line_output_type=configs.T_F32), max_frames=F)
    img_a, mask_a = bf2.empty_img(F), bf2.empty_mask()
    bf2.beamform(raw, F, line_img=li)
    bf2.scanconvert(li, F, img_a, mask_a)
    img_b, mask_b = bf.empty_img(F), bf.empty_mask()
    bf.beamform_bmode(raw, F, img_b, mask_b)
    torch.cuda.synchronize()
    assert torch.equal(img_a, img_b) and torch.equal(mask_a, mask_b)


def test_c3_bench_launch_configuration():
    """C3 as the bench times it: 32 frames per call (16 virtual frames per
    CTA, four 1024-sample depth passes with carried FIR halos, row-cut
    windows), u8 sector B-mode; frames 0 and 31 vs the oracle chain."""
    w = configs.c3(sc_output_type=configs.T_U8)
    F = 32
    raw = raw_frames(w, F)
    bf = SupraBF(w, max_frames=F)
    rf_g, y_g = run_gpu(bf, raw, F)
    img = bf.empty_img(F)
    bf.scanconvert(torch.from_numpy(y_g).cuda(), F, img)
    torch.cuda.synchronize()
    for f in (0, F - 1):
        e_rf, e_db, _, env_o = check_frame(w, raw[f].cpu().numpy(), rf_g[f], y_g[f])
        assert e_rf <= RF_TOL and e_db <= DB_TOL, (f, e_rf, e_db)
        y_o, _ = oracle.log_compress(env_o, 50.0)
        img_o, _ = oracle.scan_convert(w, y_o)
        assert np.max(np.abs(img[f].cpu().numpy().astype(int) - oracle.to_u8(img_o).astype(int))) <= 1
