"""The shared input generator: splitmix64 pinned to its published outputs; value maps exact."""
import json
import os

import numpy as np

import synthgen as sg

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_splitmix64_reference_outputs():
    g = json.load(open(os.path.join(GOLD, "splitmix64.json")))
    got = [sg.word(0, i) for i in range(4)]
    assert got == [int(x, 16) for x in g["outputs_from_state0"]]
    # vectorised path agrees with the scalar one
    assert [int(x) for x in sg.words(0, np.arange(4))] == got


def test_vector_matches_scalar_random_keys():
    for s in range(5):
        key = sg.stream_key(s * 977 + 1, sg.KIND_UPDATE, s, 2 * s)
        idx = np.array([0, 1, 17, 12345, 2**40 + 3], dtype=np.uint64)
        assert [int(x) for x in sg.words(key, idx)] == [sg.word(key, int(i)) for i in idx]


def test_value_maps_exact_and_in_range():
    idx = np.arange(20000)
    u = sg.update_values(7, 3, 1, idx, sg.DTYPE_F32)
    ints = u.astype(np.float64) * 2.0**31
    assert np.all(ints == np.round(ints)) and ints.min() >= -2**23 and ints.max() < 2**23
    b = sg.update_values(7, 3, 1, idx, sg.DTYPE_BF16)
    f = sg.bf16_bits_to_f32(b).astype(np.float64) * 2.0**14
    assert np.all(f == np.round(f)) and f.min() >= -128 and f.max() <= 127
    e = sg.update_values(7, 3, 1, idx, sg.DTYPE_F32, "exact").astype(np.float64) * 2.0**20
    assert np.all(e == np.round(e)) and np.abs(e).max() <= 1024
    w = sg.w0_values(7, idx, "exact").astype(np.float64)
    assert np.all(np.abs(w) < 0.25) and np.all(w * 2**24 == np.round(w * 2**24))
    # the top bits decide the value: same word -> same value in both dtypes' sign
    wd = sg.words(sg.stream_key(7, sg.KIND_UPDATE, 3, 1), idx)
    assert np.array_equal(((wd >> np.uint64(40)).astype(np.int64) - 2**23).astype(np.float64), ints)


def test_streams_independent():
    a = sg.update_values(1, 0, 0, np.arange(64))
    b = sg.update_values(1, 1, 0, np.arange(64))
    c = sg.update_values(1, 0, 1, np.arange(64))
    assert not np.array_equal(a, b) and not np.array_equal(a, c)


def test_presets_match_paper():
    # P:1425-1430 rate set and N1/N2/N3 probabilities; P:1416-1419 C1-C3
    assert sg.RATE_SET_BPS == tuple(int(g * 1e9 / 8) for g in (1, 2.5, 3.3, 5, 10))
    assert sg.N_PRESETS["N1"] == (0, 0, 0, 0.1, 0.9)
    assert sg.N_PRESETS["N2"] == (0, 0.1, 0.1, 0.1, 0.7)
    assert sg.N_PRESETS["N3"] == (0.5, 0, 0, 0, 0.5)
    assert sg.C_PRESETS == {"C1": (10, 2), "C2": (10, 4), "C3": (4, 2)}
    r = sg.draw_rates(3, 4000, "N1")
    frac5 = r.count(625_000_000) / len(r)
    assert set(r) <= {625_000_000, 1_250_000_000} and 0.07 < frac5 < 0.13


def test_shuffle_is_permutation():
    s = sg.shuffle(5, list(range(32)))
    assert sorted(s) == list(range(32)) and s != list(range(32))
