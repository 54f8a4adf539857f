"""C-ABI contract (CPU): the library loads, exports every symbol the header
declares, the ctypes struct matches the C layout, and parameter validation
returns the documented status before touching a device (T6)."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import numpy as np
import pytest

import paper_1711_06127_b200 as pb
from paper_1711_06127_b200 import binding
from synth import configs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "supra_bf.h")


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_1711_06127_b200 import build
    build.build()


def declared_symbols():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"\b(supra_bf_[a-z_]+)\s*\(", txt)))


def test_exports_every_declared_symbol():
    syms = declared_symbols()
    assert set(syms) == set(binding.EXPORTS)
    L = C.CDLL(binding.LIB_PATH)
    for s in syms:
        assert hasattr(L, s), s
    out = subprocess.check_output(["nm", "-D", "--defined-only", binding.LIB_PATH]).decode()
    for s in syms:
        assert re.search(rf"\bT {s}\b", out), s


def test_struct_layout_matches_header():
    fields = [f for f, _ in binding.Config._fields_]
    src = "#include <stdio.h>\n#include <stddef.h>\n#include \"supra_bf.h\"\nint main(){\n"
    src += 'printf("%zu\\n", sizeof(supra_bf_config));\n'
    for f in fields:
        src += f'printf("%zu\\n", offsetof(supra_bf_config, {f}));\n'
    src += "return 0;}\n"
    with tempfile.TemporaryDirectory() as d:
        cf = os.path.join(d, "t.c")
        open(cf, "w").write(src)
        exe = os.path.join(d, "t")
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), cf, "-o", exe])
        vals = [int(x) for x in subprocess.check_output([exe]).split()]
    assert vals[0] == C.sizeof(binding.Config)
    for f, off in zip(fields, vals[1:]):
        assert getattr(binding.Config, f).offset == off, f


def _create(w, **over):
    cfg, keep = binding.make_config(w, 0, 1, **over)
    h = C.c_void_p()
    rc = binding.lib().supra_bf_create(C.byref(cfg), C.byref(h))
    if rc == 0:
        binding.lib().supra_bf_destroy(h)
    return rc, binding.lib().supra_bf_last_error().decode()


@pytest.mark.parametrize("field,value", [
    ("speed_of_sound_mps", 999.0), ("speed_of_sound_mps", 2001.0), ("f_number", 0.0),
    ("fir_taps", 64), ("fir_taps", 0), ("dynamic_range_db", 0.0), ("samples_per_channel", 1020),
    ("pitch_x_mm", -0.3), ("window", 7), ("decimation", 0), ("decimation", 1024), ("abi_version", 99),
    ("max_frames_per_call", 0), ("demod_bandwidth_hz", 80e6), ("fov_x_deg", 180.0),
    ("interpolation", 2),
])
def test_param_errors(field, value):
    w = configs.c3() if field == "fov_x_deg" else configs.c1()
    rc, msg = _create(w, **{field: value})
    assert rc == binding.E_PARAM, (rc, msg)
    assert msg


def test_fixed_reference_must_be_positive():
    rc, _ = _create(configs.c1(), reference_mode=binding.REF_FIXED, reference_value=0.0)
    assert rc == binding.E_PARAM


def test_line_event_out_of_range_is_struct_error():
    w = configs.c1()
    ev = w.line_event.copy()
    ev[5] = 64
    rc, _ = _create(w.replace(line_event=ev))
    assert rc == binding.E_STRUCT


def test_geometry_must_match_scan_conversion():
    w = configs.c1()
    o = w.line_origin_mm.copy()
    o[3, 0] += 0.01                      # uneven linear origins
    assert _create(w.replace(line_origin_mm=o))[0] == binding.E_PARAM
    w3 = configs.c3()
    d = w3.line_direction.copy()
    d[0] = [0, 0, 1]                     # off the uniform angle grid
    assert _create(w3.replace(line_direction=d))[0] == binding.E_PARAM


def test_valid_config_without_gpu_is_cuda_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    rc, msg = _create(configs.c1())
    assert rc == binding.E_CUDA and "no CUDA device" in msg
    with pytest.raises(binding.SupraError):
        pb.SupraBF(configs.c1())


def test_null_handle_calls():
    L = binding.lib()
    assert L.supra_bf_beamform(None, None, 1, None, None, None) == binding.E_STRUCT
    assert L.supra_bf_envelope_log(None, None, 1, None, None) == binding.E_STRUCT
    assert L.supra_bf_scanconvert(None, None, 1, None, None, None) == binding.E_STRUCT
    assert L.supra_bf_stage_raw(None, None, None, 1, None, None) == binding.E_STRUCT
    L.supra_bf_destroy(None)
    assert _create.__name__  # destroy(NULL) is a no-op


@pytest.mark.parametrize("bands", [
    ((7e6, 4.2e6, 0.5), (3.5e6, 2e6, 0.4)),        # weights sum to 0.9
    ((7e6, 4.2e6, 1.2), (3.5e6, 2e6, -0.2)),       # negative weight
    ((7e6, 4.2e6, 0.5), (19.5e6, 2e6, 0.5)),       # band past fs/2
    ((7e6, 4.2e6, 0.2),) * 5,                      # more than SUPRA_MAX_BANDS
])
def test_band_bank_errors(bands):
    w = configs.c1(bands=bands)
    if len(bands) > binding.MAX_BANDS:
        with pytest.raises(ValueError):
            binding.make_config(w)
        cfg, _ = binding.make_config(configs.c1(bands=bands[:4]))
        cfg.num_bands = 5
        h = C.c_void_p()
        assert binding.lib().supra_bf_create(C.byref(cfg), C.byref(h)) == binding.E_PARAM
        return
    rc, msg = _create(w)
    assert rc == binding.E_PARAM and "band" in msg, (rc, msg)


def test_channel_map_errors():
    w = configs.table1(64, 1)
    bad = w.channel_element.copy()
    bad[5, 3] = bad[5, 4]                            # element twice in one event
    assert _create(w.replace(channel_element=bad))[0] == binding.E_STRUCT
    bad = w.channel_element.copy()
    bad[0, 0] = 128                                  # not an element
    assert _create(w.replace(channel_element=bad))[0] == binding.E_STRUCT
