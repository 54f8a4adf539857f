"""Input generator checks (harness; not under parity)."""
import numpy as np

import synth
from synth import configs


def test_empty_field_zero():
    w = configs.c1()
    sig = synth.signal_cpu(w, np.zeros((0, 4)))
    assert np.all(sig == 0.0)


def test_echo_timing_S432():
    # single on-axis scatterer at 20 mm, centred element/event: echo centre
    # at round(2 * 0.020 / 1540 * fs) = sample 1039
    o, d = configs.linear_lines(np.array([0.0]))
    w = configs.Workload("e", 1, 1, 0.3, 0.3, 7e6, 1, 2048, 1, 1, o, d, np.zeros(1, np.int32),
                         np.zeros((1, 3)), configs.SC_LINEAR_2D, (2, 1, 2), (0, 0, 0),
                         (1, 1, 1))
    sig = synth.signal_cpu(w, np.array([[0.0, 0.0, 20.0, 1.0]]))
    assert np.argmax(np.abs(sig[0, 0])) == round(2 * 0.020 / 1540 * 40e6)


def test_superposition():
    w = configs.c1().replace(S=512)
    a = np.array([[0.3, 0.0, 5.0, 1.0]])
    b = np.array([[-1.2, 0.0, 7.0, 0.5]])
    sa, sb = synth.signal_cpu(w, a), synth.signal_cpu(w, b)
    sab = synth.signal_cpu(w, np.concatenate([a, b]))
    assert np.max(np.abs(sab - sa - sb)) <= 1e-12 * np.max(np.abs(sab))


def test_quantize_headroom_and_seeded_noise():
    w = configs.c1()
    raw = synth.channel_data_cpu(w)
    assert np.max(np.abs(raw)) == 8192          # peak -> 32767/4 (12 dB headroom)
    w2 = w.replace(noise_db=-40.0)
    r1 = synth.channel_data_cpu(w2)
    r2 = synth.channel_data_cpu(w2)
    assert np.array_equal(r1, r2) and not np.array_equal(r1, raw)
