"""supra_bf_stage_raw (the end-to-end path's host->device transfer): the
device copies only the sample ranges the beamformer reads (SURVEY 8(d),
"fetch windows, not whole rows").  The rest of the destination is left as
it was -- here deliberately filled with random int16 -- so beamforming the
staged buffer must give BITWISE the RF and line image of the full buffer on
every geometry and option that changes which samples a tap reads: linear,
phased, matrix with multi-line events, a walking-aperture channel map,
nearest-sample lookup, a non-zero t0, and decimation."""
import pytest

from synth import configs

from gpu_util import raw_frames

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1711_06127_b200 import SupraBF, binding  # noqa: E402

CASES = [
    ("C1", 1, {}),
    ("C1-nearest", 1, {"interpolation": configs.INTERP_NEAREST}),
    ("C1-t0", 1, {"t0_s": 0.37e-6}),
    ("C2", 4, {}),
    ("C3", 2, {"decimation": 2}),
    ("C4b", 1, {}),
    ("T1_64_2", 3, {}),
]


def _full_and_staged(w, F, src_on_host=True):
    raw = raw_frames(w, F)
    bf = SupraBF(w, max_frames=F)
    g = torch.Generator(device="cuda").manual_seed(7)
    dst = torch.randint(-32768, 32767, raw.shape, dtype=torch.int16, device="cuda", generator=g)
    src = raw.cpu().pin_memory() if src_on_host else raw
    nbytes = bf.stage_raw(src, dst, F)
    out = []
    for buf in (raw, dst):
        rf, li = bf.empty_rf(F), bf.empty_line_img(F)
        bf.beamform(buf, F, rf=rf, line_img=li)
        out.append((rf.cpu(), li.cpu()))
    torch.cuda.synchronize()
    info = bf.info()
    bf.close()
    return out, nbytes, info, raw[0].numel() * 2


@pytest.mark.parametrize("name,F,over", CASES, ids=[c[0] for c in CASES])
def test_staged_input_beamforms_bitwise_equal(name, F, over):
    w = configs.CONFIGS[name.split("-")[0]](**over)
    (full, staged), nbytes, info, frame_bytes = _full_and_staged(w, F)
    assert torch.equal(full[0], staged[0]), name
    assert torch.equal(full[1], staged[1]), name
    # the staged bytes cover every referenced sample and stay below a frame
    assert info["referenced_bytes_per_frame"] <= nbytes <= frame_bytes


def test_stage_from_device_memory():
    w = configs.c2()
    (full, staged), _, _, _ = _full_and_staged(w, 2, src_on_host=False)
    assert torch.equal(full[1], staged[1])


def test_c2_stages_under_half_the_frame():
    # C2 (linear 128 ch, F = 1): 41 % of the samples are referenced
    w = configs.c2()
    bf = SupraBF(w, max_frames=1)
    raw = torch.zeros((1, w.num_events, w.C, w.S), dtype=torch.int16, device="cuda")
    n = bf.stage_raw(raw, torch.empty_like(raw), 1)
    bf.close()
    assert n < 0.5 * raw.numel() * 2


def test_stage_rejects_pageable_source():
    w = configs.c1()
    bf = SupraBF(w, max_frames=1)
    raw_h = torch.zeros((1, w.num_events, w.C, w.S), dtype=torch.int16)  # pageable
    dst = torch.empty(raw_h.shape, dtype=torch.int16, device="cuda")
    with pytest.raises(binding.SupraError) as ei:
        bf.stage_raw(raw_h, dst, 1)
    assert ei.value.status == binding.E_STRUCT
    bf.close()
