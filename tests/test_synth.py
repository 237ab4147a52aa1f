"""The shared seeded input generator (ARA-GEN-1): known answers, determinism, shapes."""
import numpy as np
import pytest

import oracle
from paper_1412_4556_b200 import synth


def test_splitmix64_known_answers():
    # Published SplitMix64 output sequence for initial state 0 (Steele, Lea & Flood 2014 reference code):
    # next() adds the golden gamma first, so output i is sm64(i * gamma).
    assert synth.sm64_int(0) == 0xE220A8397B1DCDAF
    assert synth.sm64_int(synth.GOLDEN) == 0x6E789E6AA1B965F4
    assert synth.sm64_int(2 * synth.GOLDEN % 2**64) == 0x06C45D188009454F


def test_numpy_matches_scalar():
    seed, s = 12345, synth.stream(synth.KIND_YET_IDS)
    got = synth.draws(seed, s, 1000, 64)
    want = [synth.draw_int(seed, s, 1000 + i) for i in range(64)]
    assert [int(v) for v in got] == want
    idx = np.array([0, 7, 2**40 + 3, 2**63 + 11], dtype=np.uint64)
    assert [int(v) for v in synth.draws_at(seed, s, idx)] == [synth.draw_int(seed, s, int(i)) for i in idx]
    for n in (1, 2, 10_000, 2_000_000, 2**32 - 1):
        r = synth.draws(seed, s, 0, 16)
        assert [int(v) for v in synth.uni_np(r, n)] == [synth.uni_int(int(x), n) for x in r]


def test_yet_ids_shape_range_determinism_and_slicing():
    a = synth.yet_ids(7, 1000, 0, 50_000)
    assert a.dtype == np.uint32 and a.min() >= 1 and a.max() <= 1000
    assert np.array_equal(a, synth.yet_ids(7, 1000, 0, 50_000))
    assert np.array_equal(a[12_345:20_000], synth.yet_ids(7, 1000, 12_345, 20_000 - 12_345))
    assert not np.array_equal(a, synth.yet_ids(8, 1000, 0, 50_000))
    # roughly uniform
    h = np.bincount(a, minlength=1001)[1:]
    assert h.min() > 20 and h.max() < 90


def test_variable_lengths_and_trial_subsets():
    cfg = synth.Config.load("V")
    off = synth.trial_offsets(cfg.seed, cfg.num_trials, cfg.kmin, cfg.kmax)
    lens = np.diff(off)
    assert lens.min() >= 800 and lens.max() <= 1500
    full = synth.make_yet(cfg, 0, 50)
    sub = synth.make_yet_trials(cfg, [3, 17, 49])
    for i, t in enumerate([3, 17, 49]):
        a = full.event_ids[int(full.offsets[t]):int(full.offsets[t + 1])]
        b = sub.event_ids[int(sub.offsets[i]):int(sub.offsets[i + 1])]
        assert np.array_equal(a, b)
    shard = synth.make_yet(cfg, 20, 30)
    assert np.array_equal(shard.event_ids, full.event_ids[int(full.offsets[20]):int(full.offsets[30])])


def test_elts_distinct_in_range_and_exact():
    ids = synth.elt_event_ids(5, 3, 10_000, 2_000_000)
    assert ids.size == 10_000 and np.unique(ids).size == 10_000
    assert ids.min() >= 1 and ids.max() <= 2_000_000
    full = synth.elt_event_ids(5, 3, 100, 100)          # saturation: every event present
    assert sorted(full.tolist()) == list(range(1, 101))
    li = synth.elt_losses(5, 3, 10_000, "integer")
    assert np.all(li >= 1) and np.all(li <= 2**28) and np.all(li == np.floor(li))
    assert np.array_equal(li.astype(np.float64).astype(np.float32), li)
    lr = synth.elt_losses(5, 3, 10_000, "real")
    assert np.all(np.isfinite(lr)) and np.all(lr > 0) and np.all(lr >= li) and np.all(lr <= li * np.float32(4 / 3) + 1)
    mu = synth.loss_mean_integer()
    assert abs(li.astype(np.float64).mean() / mu - 1) < 0.05


def test_tiny_config_trial_regimes():
    """the frozen terms give zero, linear and capped trials, each >= 10%."""
    cfg = synth.Config.load("T")
    y = oracle.ylt_for(cfg, synth.make_elts(cfg), synth.make_yet(cfg))[0]
    L3 = cfg.layers[0].agg.limit
    zero, capped = np.mean(y == 0), np.mean(y == L3)
    linear = 1 - zero - capped
    assert zero >= 0.1 and capped >= 0.1 and linear >= 0.1, (zero, linear, capped)


@pytest.mark.parametrize("name", ["T", "P", "PI", "M", "X", "V"])
def test_configs_load(name):
    cfg = synth.Config.load(name)
    assert cfg.num_trials > 0 and cfg.layers and all(l.agg.limit > 0 for l in cfg.layers)
    for l in cfg.layers:
        assert len(set(l.elts)) == len(l.elts) and max(l.elts) < cfg.num_elts
