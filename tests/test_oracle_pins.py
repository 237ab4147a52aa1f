"""Pins for the CPU oracle: hand-worked values, closed forms, invariants and brute force.

Nothing here re-types the oracle's formula and compares it with itself: every expected value is
either a golden fixture (hand-worked, cited in tests/golden/*.json), a closed form of a special
case (identity terms -> plain sum of raw lookups), or an invariant the mathematics fixes
(bounds, monotonicity, permutation, telescoping, exact power-of-two scaling).
"""
import itertools
import math

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import oracle
from ara_testutil import golden, golden_elts, golden_layer

INF = math.inf


# ------------------------------------------------------------------ financial terms
@pytest.mark.parametrize("x,r,l,want", [
    (100, 10, 1000, 90),    # SPEC.md:76 FT1 example
    (20, 30, 50, 0),        # SPEC.md:77 below retention
    (60, 0, INF, 60),       # SPEC.md:78 identity terms
    (90, 20, 120, 70),      # SPEC.md:85 FT2 example
    (150, 20, 120, 120),    # SPEC.md:86 limit clamp
    (0, 20, 120, 0),        # SPEC.md:87 zero loss
    (190, 50, 200, 140),    # SPEC.md:94 FT3 example
    (40, 50, 200, 0),
    (400, 50, 200, 200),
])
def test_clamp_examples(x, r, l, want):
    assert oracle.clamp(x, r, l) == want


def test_clamp_never_negative_zero():
    for x, r in [(0.0, 0.0), (0.0, 5.0), (3.0, 3.0), (1.0, 7.5)]:
        v = oracle.clamp(x, r, INF)
        assert v == 0.0 and math.copysign(1.0, v) == 1.0


@settings(max_examples=300, deadline=None)
@given(st.floats(0, 1e12), st.floats(0, 1e12), st.floats(1e-3, 1e13))
def test_clamp_bounded_and_monotone(x, r, l):
    v = oracle.clamp(x, r, l)
    assert 0.0 <= v <= l
    assert oracle.clamp(x * 2 + 1, r, l) >= v          # non-decreasing in the loss
    assert oracle.clamp(x, r * 2 + 1, l) <= v          # non-increasing in the retention
    if x <= r:
        assert v == 0.0


# ------------------------------------------------------------------ worked trials (golden)
@pytest.mark.parametrize("mode", [oracle.LOOKUP_BINARY, oracle.LOOKUP_LINEAR])
def test_spec_worked_trial(mode):
    g = golden("spec_trial_example.json")
    o, S, a, y = oracle.trial_detail(g["catalog_size"], g["trial"], golden_elts(g), golden_layer(g), mode)
    assert list(o) == g["occurrence_losses"]
    assert list(S) == g["prefix_sums"]
    assert list(a) == g["aggregate_net"]
    assert y == g["ylt"] == 140.0
    full = oracle.ylt(g["catalog_size"], np.array(g["trial"]), None, 1, len(g["trial"]), golden_elts(g),
                      [golden_layer(g)], lookup=mode)
    assert full[0, 0] == 140.0


@pytest.mark.parametrize("mode", [oracle.LOOKUP_BINARY, oracle.LOOKUP_LINEAR])
def test_extended_worked_example(mode):
    g = golden("extended_example.json")
    trials = g["trials"]
    ids = np.array([e for t in trials for e in t], dtype=np.uint32)
    off = np.zeros(len(trials) + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(t) for t in trials])
    y = oracle.ylt(g["catalog_size"], ids, off, len(trials), 0, golden_elts(g), [golden_layer(g)], lookup=mode)
    assert list(y[0]) == g["ylt"]
    d = g["detail"]
    o, S, a, yy = oracle.trial_detail(g["catalog_size"], d["trial"], golden_elts(g), golden_layer(g), mode)
    assert list(o) == d["occurrence_losses"] and list(S) == d["prefix_sums"] and list(a) == d["aggregate_net"]
    r = g["detail_reversed"]
    _, _, a2, y2 = oracle.trial_detail(g["catalog_size"], r["trial"], golden_elts(g), golden_layer(g), mode)
    assert list(a2) == r["aggregate_net"] and y2 == r["ylt"]   # same YLT, different a_k (order matters for a_k)


def test_identity_terms_sum_of_raw_lookups():
    g = golden("extended_example.json")
    elts = [(ids, losses, (0.0, INF)) for ids, losses, _ in golden_elts(g)]
    layer = (g["layer"]["elts"], (0.0, INF), (0.0, INF))
    _, _, _, y = oracle.trial_detail(g["catalog_size"], g["identity_terms"]["trial"], elts, layer)
    assert y == g["identity_terms"]["ylt"] == 2380.0


def test_brute_force_all_short_trials():
    """All 85 trials of length <= 3 over catalogue {1..4}: the YLT must equal FT3 of the sum of the
    hand-worked per-event occurrence losses (golden), for every ordering."""
    g = golden("extended_example.json")
    occ = {int(k): v for k, v in g["occurrence_loss_by_event"].items()}
    r3, l3 = g["layer"]["ft3"]
    trials = [list(t) for n in range(4) for t in itertools.product([1, 2, 3, 4], repeat=n)]
    assert len(trials) == 85
    ids = np.array([e for t in trials for e in t], dtype=np.uint32)
    off = np.zeros(len(trials) + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(t) for t in trials])
    for mode in (oracle.LOOKUP_BINARY, oracle.LOOKUP_LINEAR):
        y = oracle.ylt(g["catalog_size"], ids, off, len(trials), 0, golden_elts(g), [golden_layer(g)], lookup=mode)
        for t, v in zip(trials, y[0]):
            s = sum(occ[e] for e in t)
            assert v == min(max(s - r3, 0.0), l3), (t, v)


def test_empty_trial_and_no_hits():
    g = golden("extended_example.json")
    off = np.array([0, 0, 1], dtype=np.uint64)
    y = oracle.ylt(g["catalog_size"], np.array([5], np.uint32), off, 2, 0, golden_elts(g), [golden_layer(g)])
    assert list(y[0]) == [0.0, 0.0]


def test_id_out_of_range_rejected():
    g = golden("extended_example.json")
    with pytest.raises(oracle.OracleError):
        oracle.ylt(g["catalog_size"], np.array([6], np.uint32), None, 1, 1, golden_elts(g), [golden_layer(g)])
    with pytest.raises(oracle.OracleError):
        oracle.ylt(g["catalog_size"], np.array([0], np.uint32), None, 1, 1, golden_elts(g), [golden_layer(g)])


# ------------------------------------------------------------------ randomized invariants
def _rand_problem(seed, C=300, J=4, n=40, N=64, K=30, integer=True):
    rng = np.random.default_rng(seed)
    elts = []
    for j in range(J):
        ids = rng.choice(np.arange(1, C + 1), size=n, replace=False).astype(np.uint32)
        if integer:
            losses = rng.integers(1, 5000, size=n).astype(np.float32)
            terms = (float(rng.integers(0, 500)), float(rng.integers(500, 4000)) if j % 2 else INF)
        else:
            losses = (rng.random(n) * 5000 + 0.01).astype(np.float32)
            terms = (round(float(rng.random() * 500), 2), round(float(rng.random() * 4000 + 500), 2))
        elts.append((ids, losses, terms))
    yet = rng.integers(1, C + 1, size=N * K).astype(np.uint32)
    if integer:
        layer = (list(range(J)), (200.0, 6000.0), (1000.0, 20000.0))
    else:
        layer = (list(range(J)), (200.25, 6000.5), (1000.75, 20000.125))
    return C, elts, layer, yet, N, K


def _y(C, elts, layer, yet, N, K, **kw):
    return oracle.ylt(C, yet, None, N, K, elts, [layer], **kw)[0]


def test_identity_terms_random_equals_raw_sum():
    C, elts, layer, yet, N, K = _rand_problem(1)
    elts = [(i, l, (0.0, INF)) for i, l, _ in elts]
    layer = (layer[0], (0.0, INF), (0.0, INF))
    y = _y(C, elts, layer, yet, N, K)
    raw = [dict(zip(i.tolist(), l.tolist())) for i, l, _ in elts]
    for t in range(N):
        want = sum(d.get(int(e), 0.0) for e in yet[t * K:(t + 1) * K] for d in raw)
        assert y[t] == want


def test_bounds():
    C, elts, layer, yet, N, K = _rand_problem(2)
    y = _y(C, elts, layer, yet, N, K)
    assert np.all(y >= 0) and np.all(y <= layer[2][1])
    assert not np.any(np.signbit(y))
    for t in range(8):
        o, S, a, _ = oracle.trial_detail(C, yet[t * K:(t + 1) * K], elts, layer)
        assert np.all(o >= 0) and np.all(o <= layer[1][1])


@pytest.mark.parametrize("which", ["r1", "r2", "r3"])
def test_monotone_in_retentions(which):
    C, elts, layer, yet, N, K = _rand_problem(3)
    base = _y(C, elts, layer, yet, N, K)
    if which == "r1":
        elts = [(i, l, (r + 300.0, lim)) for i, l, (r, lim) in elts]
    elif which == "r2":
        layer = (layer[0], (layer[1][0] + 300.0, layer[1][1]), layer[2])
    else:
        layer = (layer[0], layer[1], (layer[2][0] + 3000.0, layer[2][1]))
    assert np.all(_y(C, elts, layer, yet, N, K) <= base)


@pytest.mark.parametrize("which", ["l1", "l2", "l3", "loss"])
def test_monotone_in_limits_and_losses(which):
    C, elts, layer, yet, N, K = _rand_problem(4)
    base = _y(C, elts, layer, yet, N, K)
    if which == "l1":
        elts = [(i, l, (r, lim * 2)) for i, l, (r, lim) in elts]
    elif which == "l2":
        layer = (layer[0], (layer[1][0], layer[1][1] * 2), layer[2])
    elif which == "l3":
        layer = (layer[0], layer[1], (layer[2][0], layer[2][1] * 2))
    else:
        elts = [(i, (l * np.float32(1.5)).astype(np.float32), t) for i, l, t in elts]
    assert np.all(_y(C, elts, layer, yet, N, K) >= base)


def test_permutation_invariance_integer_regime():
    C, elts, layer, yet, N, K = _rand_problem(5)
    base = _y(C, elts, layer, yet, N, K)
    rng = np.random.default_rng(0)
    perm = yet.reshape(N, K).copy()
    for row in perm:
        rng.shuffle(row)
    assert np.array_equal(_y(C, elts, layer, perm.reshape(-1), N, K), base)


def test_telescoping_aggregate_net():
    C, elts, layer, yet, N, K = _rand_problem(6)
    for t in range(N):
        o, S, a, y = oracle.trial_detail(C, yet[t * K:(t + 1) * K], elts, layer)
        assert a.sum() == y  # exact: integer regime
        assert np.all(a >= 0)


@pytest.mark.parametrize("integer", [True, False])
def test_power_of_two_scaling_is_exact(integer):
    C, elts, layer, yet, N, K = _rand_problem(7, integer=integer)
    base = _y(C, elts, layer, yet, N, K)
    s = lambda v: v * 2.0
    elts2 = [(i, (l * np.float32(2)).astype(np.float32), (s(r), s(lim))) for i, l, (r, lim) in elts]
    layer2 = (layer[0], (s(layer[1][0]), s(layer[1][1])), (s(layer[2][0]), s(layer[2][1])))
    assert np.array_equal(_y(C, elts2, layer2, yet, N, K), 2.0 * base)


@pytest.mark.parametrize("integer", [True, False])
def test_linear_binary_threads_entry_order_agree_bitwise(integer):
    C, elts, layer, yet, N, K = _rand_problem(8, integer=integer)
    base = _y(C, elts, layer, yet, N, K, threads=1)
    assert np.array_equal(_y(C, elts, layer, yet, N, K, lookup=oracle.LOOKUP_LINEAR, threads=1), base)
    assert np.array_equal(_y(C, elts, layer, yet, N, K, threads=5), base)
    rng = np.random.default_rng(1)
    shuffled = []
    for i, l, t in elts:
        p = rng.permutation(i.size)
        shuffled.append((i[p], l[p], t))
    assert np.array_equal(_y(C, shuffled, layer, yet, N, K), base)


def test_single_elt_textbook_excess_of_loss():
    """One ELT, identity FT1/FT2, FT3 = (R, L): YLT = min(max(sum of raw losses - R, 0), L)."""
    C, elts, layer, yet, N, K = _rand_problem(9)
    ids, losses, _ = elts[0]
    e = [(ids, losses, (0.0, INF))]
    R, L = 20000.0, 30000.0
    y = _y(C, e, ([0], (0.0, INF), (R, L)), yet, N, K)
    lut = np.zeros(C + 1)
    lut[ids] = losses
    raw = lut[yet].reshape(N, K).sum(axis=1)
    assert np.array_equal(y, np.minimum(np.maximum(raw - R, 0.0), L))


def test_multi_layer_rows_are_independent():
    C, elts, layer, yet, N, K = _rand_problem(10)
    l2 = (layer[0][:2], (0.0, INF), (0.0, INF))
    both = oracle.ylt(C, yet, None, N, K, elts, [layer, l2])
    assert np.array_equal(both[0], _y(C, elts, layer, yet, N, K))
    assert np.array_equal(both[1], _y(C, elts, l2, yet, N, K))


# ------------------------------------------------------------------ metrics (readings c11-c14)
def test_metric_examples_1_to_10():
    g = golden("metrics_examples.json")
    y = np.array(g["losses_1to10"], dtype=np.float64)
    for rp, want in g["pml_1to10"].items():
        assert oracle.pml(y, [float(rp)])[0] == want
    for rp, want in g["tvar_1to10"].items():
        assert oracle.tvar(y, [float(rp)])[0] == want


def test_metric_examples_8_trials():
    g = golden("metrics_examples.json")
    y = np.array(g["ylt_8trial"])
    assert [oracle.rank(8, r) for r in g["rps_8trial"]] == g["k_8trial"]
    assert list(oracle.pml(y, g["rps_8trial"])) == g["pml_8trial"]
    tv = oracle.tvar(y, g["rps_8trial"])
    assert list(tv) == [n / k for n, k in zip(g["tvar_8trial_num"], g["k_8trial"])]


def test_rank_rules():
    assert oracle.rank(1_000_000, 1000) == 1000      # alpha-form ceil((1-0.999)*N) would give 1001
    assert oracle.rank(100, 100) == 1
    assert oracle.rank(10, 2) == 5 and oracle.rank(11, 2) == 6
    assert oracle.rank(8, 8 / 3) == 3                # fuzzed ceil for non-integral RP
    for bad in (1.0, 0.5, 11.0, float("nan"), INF):
        assert oracle.rank(10, bad) == 0
    with pytest.raises(oracle.OracleError):
        oracle.pml(np.arange(10.0), [11.0])


def test_metric_invariants():
    rng = np.random.default_rng(3)
    y = np.floor(rng.exponential(1000.0, size=1000)) * (rng.random(1000) > 0.3)
    rps = [2.0, 5.0, 10.0, 20.0, 25.0, 50.0, 100.0, 200.0, 250.0, 500.0, 1000.0]
    p, t = oracle.pml(y, rps), oracle.tvar(y, rps)
    assert np.all(np.diff(p) >= 0)                   # PML non-decreasing in RP
    assert np.all(t >= p)                            # TVaR >= PML
    perm = rng.permutation(y)
    assert np.array_equal(oracle.pml(perm, rps), p) and np.array_equal(oracle.tvar(perm, rps), t)
    dup = np.concatenate([y, y])                     # N/RP integral for every RP here
    assert np.array_equal(oracle.pml(dup, rps), p)
    assert np.allclose(oracle.tvar(dup, rps), t, rtol=1e-15, atol=0)
    c = np.full(50, 7.5)
    assert np.all(oracle.pml(c, [2.0, 50.0]) == 7.5) and np.all(oracle.tvar(c, [2.0, 50.0]) == 7.5)


# ------------------------------------------------------------------ N4 outputs: OLT (occurrence basis), AAL, EP
def test_olt_extended_example():
    g = golden("extended_example.json")
    trials = g["trials"]
    ids = np.array([e for t in trials for e in t], dtype=np.uint32)
    off = np.zeros(len(trials) + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(t) for t in trials])
    y, o = oracle.ylt_olt(g["catalog_size"], ids, off, len(trials), 0, golden_elts(g), [golden_layer(g)])
    assert list(y[0]) == g["ylt"] and list(o[0]) == g["olt"]


def test_olt_bounds_and_relation_to_ylt():
    C, elts, layer, yet, N, K = _rand_problem(11)
    y, o = oracle.ylt_olt(C, yet, None, N, K, elts, [layer])
    assert np.all(o >= 0) and np.all(o <= layer[1][1])           # occurrence losses are within FT2's limit
    ident = (layer[0], layer[1], (0.0, INF))
    s, _ = oracle.ylt_olt(C, yet, None, N, K, elts, [ident])
    assert np.all(o <= s)                                          # the largest occurrence <= the trial sum
    assert np.array_equal(y, oracle.ylt(C, yet, None, N, K, elts, [layer]))


def test_aal_and_ep_examples():
    g = golden("metrics_examples.json")
    assert oracle.aal(np.arange(1, 11.0)) == g["aal_1to10"]
    assert list(oracle.ep(np.array(g["ep_losses"]), g["ep_thresholds"])) == g["ep_probs"]
    y = np.array([0.0, 5.0, 5.0, 7.0])
    assert oracle.aal(y) == 4.25 and list(oracle.ep(y, [5.0, 5.1, 0.0])) == [0.75, 0.25, 1.0]


def test_layer_totals_hand_worked():
    """Program / portfolio totals, worked by hand: three layers, two groups.
    The third trial pins the summation order (layer order): fl(fl(1e16 + 1) + 1) = 1e16 (ulp(1e16) = 2,
    ties to even), whereas summing the two 1's first would give 1e16 + 2."""
    ylt = np.array([[1.0, 2.0, 1e16],
                    [10.0, 20.0, 7.0],
                    [100.0, 200.0, 1.0],
                    [0.0, 0.5, 1.0]])
    group = [0, 1, 0, 0]
    got = oracle.layer_totals(ylt, group, 2)
    assert np.array_equal(got, np.array([[101.0, 202.5, 1e16],
                                         [10.0, 20.0, 7.0]]))
    assert 1e16 + 2.0 != 1e16  # the alternative order is distinguishable
    # a group with no layer is all zero; one group is the column sum of a small integer matrix
    assert np.array_equal(oracle.layer_totals(ylt[:2, :2], [1, 1], 3), np.array([[0.0, 0.0], [11.0, 22.0], [0.0, 0.0]]))
