"""GPU parity for every launch shape bench.py times, and batch invariance.

Each bench line runs a DAS launch shape (frames per CTA x tiles per pass)
that these tests run too, on the same workload, against the binary64 oracle
(SURVEY 8(c)); gates as in test_parity_gpu.py (north_star: RF normwise
<= 1e-4, <= 0.01 dB on the log-compressed image).  3D volumes are compared
on sampled scanlines -- the oracle costs ~70 ms per C4 line per core -- with
a FIXED log reference taken from the oracle's envelope, so the fused line
image of the sampled lines is comparable line by line.

Shapes: whatever pick_shape (csrc/host.cpp) chooses for the bench's call --
frames per CTA x tiles per pass x mirror lines per CTA:
  C2 100 frames        <16,4> + remainder launch   (headline)
  C4b 8 volumes        mirror lines, 8-volume batch (bench C4b_stream)
  C4p 4 volumes        S = 3648, mirror pairs       (bench C4p_stream)
  C4a / C4b 1 volume   mirror quads <1,8,MIR=4>     (bench C4a_single, C4b_single)
  C4p 1 volume         mirror pairs <1,16,MIR=2>    (bench C4p_single)
  T1 64 frames         <16,4>, S = 2368 (3rd pass partial)   (bench T1_*)
  PSF 1 frame          linear, single frame, S = 1408 (tests/test_psf_gpu.py)
Every shape sums each output's members in the same fixed order (DESIGN
reading B6), so results do not depend on the shape; the batch-invariance
tests below check that bitwise.
"""
import numpy as np
import pytest

import oracle
import synth
from synth import configs

from gpu_util import DB_TOL, RF_TOL, db_err, oracle_chain, raw_frames, rf_err, run_gpu

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1711_06127_b200 import SupraBF  # noqa: E402


def distinct_volumes(w, n):
    """n volumes, volume v = realisation v (distinct noise), on the device."""
    out = torch.empty((n, w.num_events, w.C, w.S), dtype=torch.int16, device="cuda")
    for v in range(n):
        synth.channel_data_gpu(w, out[v], realisation=v)
    torch.cuda.synchronize()
    return out


def sampled_fixed_ref_parity(w, raw, vols, lines, check_vols):
    """Run the bench's launch (all ``vols`` volumes in one call) with a fixed
    reference from the oracle's envelope and RF output, and compare the
    sampled lines of ``check_vols`` with the oracle chain."""
    envs = {}
    for v in check_vols:
        rf_o, env_o = oracle_chain(w, raw[v].cpu().numpy(), lines=lines)
        envs[v] = (rf_o, env_o)
    ref = max(float(e.max()) for _, e in envs.values())
    wf = w.replace(reference_mode=configs.REF_FIXED, reference_value=ref,
                   line_output_type=configs.T_F32)
    bf = SupraBF(wf, max_frames=vols)
    rf = bf.empty_rf(vols)
    li = bf.empty_line_img(vols)
    bf.beamform(raw, vols, rf=rf, line_img=li)
    torch.cuda.synchronize()
    worst = (0.0, 0.0)
    for v, (rf_o, env_o) in envs.items():
        e_rf = rf_err(rf[v].cpu().numpy()[lines], rf_o)
        y_o, _ = oracle.log_compress(env_o, w.dynamic_range_db, ref_mode=1, ref_value=ref)
        e_db = db_err(li[v].cpu().numpy()[lines], y_o, w.dynamic_range_db)
        assert e_rf <= RF_TOL, (v, e_rf)
        assert e_db <= DB_TOL, (v, e_db)
        worst = (max(worst[0], e_rf), max(worst[1], e_db))
    bf.close()
    return worst


def c4_lines(w, seed, n=10):
    rng = np.random.default_rng(seed)
    L = w.L
    fixed = [0, L // 2 - 1, L // 2 + w.num_lines_x // 2, L - 1]
    return np.sort(np.unique(np.concatenate([fixed, rng.choice(L, n, replace=False)]))).astype(np.int32)


# ------------------------------------------------------------ 3D launch shapes
def test_c4b_stream_shape_8_volumes():
    w = configs.c4("b")
    raw = distinct_volumes(w, 8)
    sampled_fixed_ref_parity(w, raw, 8, c4_lines(w, 21), check_vols=(0, 5, 7))


def test_c4a_stream_shape_2_volumes_and_batch_invariance():
    # bench C4a_stream: two 16 GiB volumes per call (mirror quads, 2 volumes
    # per CTA); the oracle on sampled lines of both, and each volume's RF and
    # line image bitwise equal to its own single-volume call (reading B6)
    w = configs.c4("a")
    raw = distinct_volumes(w, 2)
    sampled_fixed_ref_parity(w, raw, 2, c4_lines(w, 25, n=6), check_vols=(0, 1))
    bf = SupraBF(w, max_frames=2)
    rf2, li2 = bf.empty_rf(2), bf.empty_line_img(2)
    bf.beamform(raw, 2, rf=rf2, line_img=li2)
    for v in range(2):
        rf1, li1 = bf.empty_rf(1), bf.empty_line_img(1)
        bf.beamform(raw[v:v + 1], 1, rf=rf1, line_img=li1)
        torch.cuda.synchronize()
        assert torch.equal(rf1[0], rf2[v]), v
        assert torch.equal(li1[0], li2[v]), v
        del rf1, li1
    bf.close()


@pytest.mark.parametrize("variant", ["a", "b"])
def test_c4_single_volume_fused_line_image(variant):
    # one volume per call (mirror quads) with the fused envelope/log epilogue
    w = configs.c4(variant)
    raw = distinct_volumes(w, 1)
    sampled_fixed_ref_parity(w, raw, 1, c4_lines(w, 22), check_vols=(0,))


def test_c4p_stream_shape_4_volumes():
    w = configs.c4p()
    raw = distinct_volumes(w, 4)
    sampled_fixed_ref_parity(w, raw, 4, c4_lines(w, 23, n=8), check_vols=(0, 3))


def test_c4p_single_volume_fused_line_image():
    w = configs.c4p()
    raw = distinct_volumes(w, 1)
    sampled_fixed_ref_parity(w, raw, 1, c4_lines(w, 24, n=8), check_vols=(0,))


# ------------------------------------------------------------ 2D launch shapes
@pytest.mark.parametrize("E,M", [(64, 1), (128, 2)])
def test_table1_bench_launch_64_frames(E, M):
    # S = 2368: two full 1024-sample passes and a 320-sample third pass
    w = configs.table1(E, M, sc_output_type=configs.T_U8)
    F = 64
    raw = raw_frames(w, F)
    bf = SupraBF(w, max_frames=F)
    rf_g, y_g = run_gpu(bf, raw, F)
    img = bf.empty_img(F)
    bf.scanconvert(torch.from_numpy(y_g).cuda(), F, img)
    torch.cuda.synchronize()
    for f in (0, 37, 63):
        rf_o, env_o = oracle_chain(w, raw[f].cpu().numpy())
        assert rf_err(rf_g[f], rf_o) <= RF_TOL, f
        y_o, _ = oracle.log_compress(env_o, w.dynamic_range_db)
        assert db_err(y_g[f], y_o) <= DB_TOL, f
        img_o, _ = oracle.scan_convert(w, y_o)
        got = img[f].cpu().numpy().astype(int)
        assert np.max(np.abs(got - oracle.to_u8(img_o).astype(int))) <= 1, f


def test_psf_wire_phantom_launch_vs_oracle():
    # tests/test_psf_gpu.py's launch: one frame, S = 1408 (<1,8>), through
    # beamform_lines (DAS + envelope, pre-log) and the fused beamform
    w = configs.psf_linear()
    raw = torch.empty((1, w.num_events, w.C, w.S), dtype=torch.int16, device="cuda")
    synth.channel_data_gpu(w, raw[0], scat=configs.wire_phantom((5.0, 10.0, 15.0, 20.0, 25.0)))
    torch.cuda.synchronize()
    bf = SupraBF(w)
    env = torch.zeros((1, w.L, w.S), dtype=torch.float32, device="cuda")
    fmax = torch.zeros((1,), dtype=torch.float32, device="cuda")
    bf.beamform_lines(raw, 1, 0, w.L, env, fmax)
    rf_g, y_g = run_gpu(bf, raw, 1)
    rf_o, env_o = oracle_chain(w, raw[0].cpu().numpy())
    assert rf_err(rf_g[0], rf_o) <= RF_TOL
    e = env[0].cpu().numpy().astype(np.float64)
    assert np.max(np.abs(e - env_o)) / np.max(env_o) <= RF_TOL
    assert abs(float(fmax[0]) - env_o.max()) / env_o.max() <= RF_TOL
    y_o, _ = oracle.log_compress(env_o, w.dynamic_range_db)
    assert db_err(y_g[0], y_o) <= DB_TOL


# ------------------------------------------------------------ batch invariance
def _frames_of(bf, raw, F):
    rf = bf.empty_rf(F)
    li = bf.empty_line_img(F)
    bf.beamform(raw, F, rf=rf, line_img=li)
    torch.cuda.synchronize()
    return rf, li


def test_batch_invariance_bitwise_c2():
    """A frame's RF and line image are bitwise the same whatever call it is
    beamformed in (supra_bf.h "Results are deterministic"): 100
    frames (<16,4> + <4,8> remainder), 16, 8 (<8,8>), 3 (<2,x> + a 1-frame
    remainder in the batch kernel), 2.  A 1-frame call (warp-split kernel)
    agrees to float32 rounding."""
    w = configs.c2()
    F = 100
    raw = raw_frames(w, F)
    for f in range(F):              # make every frame distinct
        if f >= 4:
            raw[f] = torch.roll(raw[f], shifts=f, dims=-1)
    bf = SupraBF(w, max_frames=F)
    rf100, li100 = _frames_of(bf, raw, F)
    for F2, off in ((16, 83), (8, 90), (3, 97), (2, 50), (17, 40)):
        rf2, li2 = _frames_of(bf, raw[off:off + F2], F2)
        assert torch.equal(rf2, rf100[off:off + F2]), (F2, off)
        assert torch.equal(li2, li100[off:off + F2]), (F2, off)
    rf1, li1 = _frames_of(bf, raw[98:99], 1)
    a = rf1[0].cpu().numpy().astype(np.float64)
    b = rf100[98].cpu().numpy().astype(np.float64)
    assert rf_err(a, b) <= 1e-6
    # (RF within 1e-6 of the frame max moves a pixel at the -50 dB floor by
    # up to 8.7 x 1e-6 / 10^(-50/20) = 2.8e-3 dB)
    assert db_err(li1[0].cpu().numpy(), li100[98].cpu().numpy().astype(np.float64)) <= 5e-3
    # one frame against the oracle, from the 100-frame call
    rf_o, env_o = oracle_chain(w, raw[97].cpu().numpy())
    assert rf_err(rf100[97].cpu().numpy(), rf_o) <= RF_TOL


def test_batch_invariance_bitwise_c3():
    # S = 4096: four 1024-sample passes at 16 frames, <2,16> / <4,16> at 2-4 frames
    w = configs.c3()
    raw = raw_frames(w, 16)
    for f in range(1, 16):
        raw[f] = torch.roll(raw[0], shifts=3 * f, dims=-1)
    bf = SupraBF(w, max_frames=16)
    rf16, li16 = _frames_of(bf, raw, 16)
    for F2, off in ((4, 12), (2, 7), (5, 3)):
        rf2, li2 = _frames_of(bf, raw[off:off + F2], F2)
        assert torch.equal(rf2, rf16[off:off + F2]), (F2, off)
        assert torch.equal(li2, li16[off:off + F2]), (F2, off)


# ------------------------------------------------------------ e2e path
def test_host_pipeline_equals_device_calls():
    """HostPipeline (the e2e path bench.py times: pinned host frames -> H2D ->
    beamform + scanconvert on two streams -> D2H) gives bitwise the images of
    the device calls on the same frames."""
    from paper_1711_06127_b200.pipeline import HostPipeline
    w = configs.c2(sc_output_type=configs.T_U8)
    F = 16
    raw = raw_frames(w, F)
    bf = SupraBF(w, max_frames=F)
    li = bf.empty_line_img(F)
    img = bf.empty_img(F)
    bf.beamform(raw, F, line_img=li)
    bf.scanconvert(li, F, img)
    torch.cuda.synchronize()
    raw_h = raw.cpu().pin_memory()
    nx, ny, nz = w.out_dims
    img_h = torch.empty((F, nz, ny, nx), dtype=torch.uint8).pin_memory()
    HostPipeline(bf, chunk=4).run(raw_h, img_h)
    assert torch.equal(img_h, img.cpu())


# ------------------------------------------------------------ indices with decimation
def test_sector_decimation_sc_indices():
    # supra_bf_sc_indices decodes the (decimated) line-image index: k0 < S/d
    w = configs.c3(decimation=2)
    bf = SupraBF(w)
    valid_o, idx_o, _ = oracle.sc_table(w)
    valid_g, idx_g = bf.sc_indices()
    assert np.array_equal(valid_g, valid_o)
    v = valid_o.astype(bool)
    assert np.array_equal(idx_g[v], idx_o[v])
    assert idx_g[v][:, 2].max() < w.S // 2


# ----------------- linear scan conversion from a u8 line image (the bench's
# Table-1 lines): the 2-D tensor copy stages the bytes (a quarter of the f32
# slab), the depth lerp reads y = v / 255.
@pytest.mark.parametrize("name,F", [("C2", 3), ("T1_64_1", 5)])
def test_linear_sc_u8_line_image(name, F):
    w8 = configs.CONFIGS[name]().replace(line_output_type=configs.T_U8, sc_output_type=configs.T_F32)
    g = torch.Generator().manual_seed(7)
    L, S = w8.L, w8.S
    li8 = torch.randint(0, 256, (F, L, S), generator=g, dtype=torch.uint8)
    bf8 = SupraBF(w8, max_frames=F)
    img = bf8.empty_img(F)
    mask = bf8.empty_mask()
    bf8.scanconvert(li8.cuda(), F, img, mask)
    # the same values as an f32 line image (v * fl(1/255) in f32, the
    # kernel's own conversion): the f32 path must give the same bits
    wf = w8.replace(line_output_type=configs.T_F32)
    bff = SupraBF(wf, max_frames=F)
    lif = (li8.to(torch.float32) * torch.tensor(1.0 / 255.0, dtype=torch.float32)).cuda()
    imgf = bff.empty_img(F)
    bff.scanconvert(lif, F, imgf)
    torch.cuda.synchronize()
    assert torch.equal(img, imgf)
    # vs the oracle (binary64) on the first and last frame
    for f in (0, F - 1):
        img_o, mask_o = oracle.scan_convert(w8, li8[f].numpy().astype(np.float64) / 255.0)
        assert np.array_equal(mask.cpu().numpy().reshape(mask_o.shape), mask_o)
        assert db_err(img.cpu().numpy()[f].reshape(img_o.shape), img_o) <= DB_TOL
    # u8 B-mode from the u8 line image: within one LSB of the oracle
    wu = w8.replace(sc_output_type=configs.T_U8)
    bfu = SupraBF(wu, max_frames=F)
    imgu = bfu.empty_img(F)
    bfu.scanconvert(li8.cuda(), F, imgu)
    img_o, _ = oracle.scan_convert(wu, li8[F - 1].numpy().astype(np.float64) / 255.0)
    d = imgu.cpu().numpy()[F - 1].reshape(img_o.shape).astype(int) - oracle.to_u8(img_o).astype(int)
    assert np.max(np.abs(d)) <= 1
    for b in (bf8, bff, bfu):
        b.close()


# -------- records that are not a multiple of the pass length: the first pass
# starts at S - ceil(S/PL) PL < 0 and holds the remainder,
# down to a single 32-sample row of real samples (S = 1056 with 1024-sample
# passes); results vs the oracle and bitwise across launch shapes.
@pytest.mark.parametrize("S", [1056, 1312, 2080])
def test_short_first_pass(S):
    w = configs.c1(S=S)
    raw = torch.empty((16, w.num_events, w.C, w.S), dtype=torch.int16, device="cuda")
    for f in range(16):
        synth.channel_data_gpu(w, raw[f], realisation=f % 4)
    torch.cuda.synchronize()
    bf = SupraBF(w, max_frames=16)
    rf16, y16 = run_gpu(bf, raw, 16)
    rf6, y6 = run_gpu(bf, raw, 6)
    rf1, y1 = run_gpu(bf, raw, 1)
    assert np.array_equal(rf16[:6], rf6) and np.array_equal(y16[:6], y6)
    for f in (0, 5):
        rf_o, env_o = oracle_chain(w, raw[f].cpu().numpy())
        assert rf_err(rf16[f], rf_o) <= RF_TOL
        y_o, _ = oracle.log_compress(env_o, w.dynamic_range_db, w.reference_mode, w.reference_value)
        assert db_err(y16[f], y_o) <= DB_TOL
    rf_o, env_o = oracle_chain(w, raw[0].cpu().numpy())
    assert rf_err(rf1[0], rf_o) <= RF_TOL
    bf.close()


# ----------------- table scan conversion (sector 2D, pyramid 3D) from a u8
# line image, the bench's 3D lines: the row-walking kernel blends the bytes
# as integers and scales by 1/255 once; vs the oracle on y = v / 255.
@pytest.mark.parametrize("name,F", [("C3", 3), ("C4b", 1)])
def test_table_sc_u8_line_image(name, F):
    w = configs.CONFIGS[name]().replace(line_output_type=configs.T_U8, sc_output_type=configs.T_F32)
    g = torch.Generator().manual_seed(11)
    li8 = torch.randint(0, 256, (F, w.L, w.S), generator=g, dtype=torch.uint8)
    bf = SupraBF(w, max_frames=F)
    img, mask = bf.empty_img(F), bf.empty_mask()
    bf.scanconvert(li8.cuda(), F, img, mask)
    wu = w.replace(sc_output_type=configs.T_U8)
    bfu = SupraBF(wu, max_frames=F)
    imgu = bfu.empty_img(F)
    bfu.scanconvert(li8.cuda(), F, imgu)
    torch.cuda.synchronize()
    f = F - 1
    img_o, mask_o = oracle.scan_convert(w, li8[f].numpy().astype(np.float64) / 255.0)
    assert np.array_equal(mask.cpu().numpy().reshape(mask_o.shape), mask_o)
    assert db_err(img.cpu().numpy()[f].reshape(img_o.shape), img_o) <= DB_TOL
    d = imgu.cpu().numpy()[f].reshape(img_o.shape).astype(int) - oracle.to_u8(img_o).astype(int)
    assert np.max(np.abs(d)) <= 1
    bf.close()
    bfu.close()
