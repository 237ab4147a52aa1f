"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Tolerance (north_star): |gpu - oracle| <= max(1e-6 |oracle|, 1e-3) for the real regime; BITWISE in
the integer regime, where every fp64 operation of both paths is exact, and for
the hand-worked golden values.  Inputs come from the shared generator (synth) or the golden files;
no oracle input or expected value is ever produced by the CUDA path.
"""
import math

import numpy as np
import pytest
import torch

import oracle
from ara_testutil import (KERNEL_STREAM, gpu_ylt, golden, golden_context, golden_elts, golden_layer, ragged, select,
                          variants, within_tol)
from paper_1412_4556_b200 import ara, synth

pytestmark = pytest.mark.gpu
INF = math.inf


def _oracle_cfg(cfg, elts, yet):
    return oracle.ylt_for(cfg, elts, yet)


# ------------------------------------------------------------------ generator
def test_device_generator_matches_host(cuda_device):
    for C, q0, n in [(10_000, 0, 100_003), (2_000_000, 123_456_789, 65_536), (10_000_000, 7_999_999_000, 4099),
                     (1, 0, 17), (2**32 - 1, 2**40, 1000)]:
        out = torch.empty(n, dtype=torch.int32, device=cuda_device)
        synth.yet_ids_device(out.data_ptr(), synth.SEED, C, q0, n, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        got = out.cpu().numpy().view(np.uint32)
        assert np.array_equal(got, synth.yet_ids(synth.SEED, C, q0, n)), (C, q0, n)


# ------------------------------------------------------------------ table build (A0)
def test_table_rows_exhaustive_tiny(cuda_device):
    cfg = synth.Config.load("T")
    elts = synth.make_elts(cfg)
    ctx = ara.context_for_config(cfg, elts)
    info = ctx.ara_layer_info(0)
    assert info["table_bytes"] == 80008 and info["row_stride"] == 8
    want = np.zeros((cfg.catalog_size + 1, 2), np.float32)
    for m, j in enumerate(cfg.layers[0].elts):
        want[elts[j].event_ids, m] = elts[j].losses
    for e in range(cfg.catalog_size + 1):
        assert np.array_equal(ctx.ara_table_row(0, e), want[e]), e
    assert np.count_nonzero(want == 0) == 2 * (cfg.catalog_size + 1) - 2 * cfg.entries_per_elt
    # the test-only library's error contract (include/ara_testing.h)
    with pytest.raises(ara.AraError) as ei:
        ctx.ara_table_row(0, cfg.catalog_size + 1)
    assert ei.value.status == ara.ARA_E_RANGE
    with pytest.raises(ara.AraError) as ei:
        ctx.ara_table_row(1, 0)
    assert ei.value.status == ara.ARA_E_ARG


# ------------------------------------------------------------------ golden worked examples (bitwise)
def test_spec_worked_trial_gpu(cuda_device):
    g = golden("spec_trial_example.json")
    ctx = golden_context(g)
    y = gpu_ylt(None, ctx, np.array(g["trial"]), K=len(g["trial"]), num_trials=1)
    assert y[0, 0] == 140.0


def test_extended_example_gpu(cuda_device):
    g = golden("extended_example.json")
    ctx = golden_context(g)
    ids, off = ragged(g["trials"])
    y = gpu_ylt(None, ctx, ids, offsets_np=off)
    assert list(y[0]) == g["ylt"]
    ctx2 = golden_context(g, layers_override=[ara.Layer(g["layer"]["elts"])])
    elts_id = [ara.Elt(np.array(e["ids"], np.uint32), np.array(e["losses"], np.float32)) for e in g["elts"]]
    ctx2 = ara.Context(g["catalog_size"], elts_id, [ara.Layer(g["layer"]["elts"])])
    y2 = gpu_ylt(None, ctx2, np.array(g["identity_terms"]["trial"]), K=5, num_trials=1)
    assert y2[0, 0] == 2380.0


def test_brute_force_short_trials_gpu(cuda_device):
    import itertools
    g = golden("extended_example.json")
    trials = [list(t) for n in range(4) for t in itertools.product([1, 2, 3, 4], repeat=n)]
    ids, off = ragged(trials)
    want = oracle.ylt(g["catalog_size"], ids, off, len(trials), 0, golden_elts(g), [golden_layer(g)])
    y = gpu_ylt(None, golden_context(g), ids, offsets_np=off)
    assert np.array_equal(y, want)


# ------------------------------------------------------------------ configs
def test_tiny_config_bitwise_all_variants_and_shapes(cuda_device):
    cfg = synth.Config.load("T")
    elts = synth.make_elts(cfg)
    yet = synth.make_yet(cfg)
    want = _oracle_cfg(cfg, elts, yet)
    ctx = ara.context_for_config(cfg, elts)
    for k, v in variants(ctx):
        for bt in (64, 256):
            y = gpu_ylt(cfg, ctx, yet.event_ids, K=cfg.kmin, kernel=k, variant=v, block_threads=bt)
            assert np.array_equal(y, want), (k, v, bt)
    assert not np.any(np.signbit(y))


def test_variable_length_config_within_tolerance(cuda_device):
    cfg = synth.Config.load("V")
    elts = synth.make_elts(cfg)
    yet = synth.make_yet(cfg)
    want = _oracle_cfg(cfg, elts, yet)
    ctx = ara.context_for_config(cfg, elts)
    y = gpu_ylt(cfg, ctx, yet.event_ids, offsets_np=yet.offsets)
    assert np.all(within_tol(y, want))
    # metrics of each path's own YLT
    rps = synth.return_periods(cfg.num_trials)
    p, t = ara.ara_pml_tvar(torch.from_numpy(y[0]).cuda(), rps)
    assert np.all(within_tol(p, oracle.pml(want[0], rps))) and np.all(within_tol(t, oracle.tvar(want[0], rps)))


def _small_problem(J, C=5000, n=300, K=37, N=333, integer=True, seed=0, inf_limits=False, zero_ret=False,
                   empty_elts=()):
    rng = np.random.default_rng(seed + 1000 * J)
    elts = []
    for j in range(J):
        cnt = 0 if j in empty_elts else n
        ids = rng.choice(np.arange(1, C + 1), size=cnt, replace=False).astype(np.uint32)
        losses = (rng.integers(1, 1 << 20, size=cnt) if integer else rng.random(cnt) * 1e6 + 0.5).astype(np.float32)
        r = 0.0 if zero_ret else float(rng.integers(0, 1 << 18))
        l = INF if (inf_limits or j % 3 == 1) else float(rng.integers(1 << 18, 1 << 21))
        elts.append((ids, losses, (r, l)))
    # ids 1 and C present
    yet = rng.integers(1, C + 1, size=N * K).astype(np.uint32)
    yet[0], yet[-1] = 1, C
    layer = (list(range(J)), (0.0 if zero_ret else 5000.0, INF if inf_limits else float(1 << 22)),
             (0.0 if zero_ret else 2e5, INF if inf_limits else 4e6))
    return C, elts, layer, yet, N, K


def _ctx_from(C, elts, layers):
    return ara.Context(C, [ara.Elt(i, l, r, lim) for i, l, (r, lim) in elts],
                       [ara.Layer(idx, a[0], a[1], b[0], b[1]) for idx, a, b in layers])


@pytest.mark.parametrize("J", [1, 2, 3, 4, 5, 8, 9, 15, 16, 17, 24, 31, 33, 64, 100, 128])
def test_every_row_width_bitwise(cuda_device, J):
    C, elts, layer, yet, N, K = _small_problem(J)
    want = oracle.ylt(C, yet, None, N, K, elts, [layer])
    ctx = _ctx_from(C, elts, [layer])
    for k, v in variants(ctx):
        assert np.array_equal(gpu_ylt(None, ctx, yet, K=K, kernel=k, variant=v), want), (k, v)


@pytest.mark.parametrize("J", [2, 16, 100])
def test_exact_filter_stage_bitwise(cuda_device, J):
    """ARA_OPT_FILTER: with a folded bitmap (3M-event catalogue > the shared-memory bitmap) the exact filter
    stage fetches records only for true hits and gives false positives a zero record; the YLT (and the
    occurrence loss table) must equal the oracle bitwise with the stage forced on, forced off and auto, for
    fixed and ragged trials.  Also forced on for an unfolded bitmap."""
    for C, n in ((3_000_000, 20_000), (5000, 300)):
        Cc, elts, layer, yet, N, K = _small_problem(J, C=C, n=n, K=1000 if C > 5000 else 37,
                                                    N=300 if C > 5000 else 333)
        want = oracle.ylt(Cc, yet, None, N, K, elts, [layer])
        rng = np.random.default_rng(J)
        lens = rng.integers(0, 1500, size=200)
        off = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
        ryet = yet[: int(off[-1])] if off[-1] <= yet.size else np.resize(yet, int(off[-1]))
        rwant = oracle.ylt(Cc, ryet, off, len(lens), 0, elts, [layer])
        ctx = _ctx_from(Cc, elts, [layer])
        ctx.ara_set_option(ara.ARA_OPT_KERNEL, ara.KERNEL_PRESENCE)
        for f in (1, 0, -1):
            ctx.ara_set_option(ara.ARA_OPT_FILTER, f)
            assert np.array_equal(gpu_ylt(None, ctx, yet, K=K), want), (C, f)
            assert np.array_equal(gpu_ylt(None, ctx, ryet, offsets_np=off), rwant), (C, f, "ragged")
        ctx.ara_set_option(ara.ARA_OPT_FILTER, 1)
        dev = torch.device("cuda:0")
        ids = torch.from_numpy(yet.view(np.int32)).to(dev)
        ylt = torch.empty((1, N), dtype=torch.float64, device=dev)
        olt = torch.empty((1, N), dtype=torch.float64, device=dev)
        ctx.ara_run_ex(ids, ylt, olt, events_per_trial=K, num_trials=N)
        ctx.ara_check()
        assert np.array_equal(ylt.cpu().numpy(), want)
        assert np.array_equal(olt.cpu().numpy(), oracle.ylt_olt(Cc, yet, None, N, K, elts, [layer])[1]), (C, "olt")
        ctx.close()


@pytest.mark.parametrize("J", [1, 2, 16, 17, 100])
def test_precombined_table_bitwise(cuda_device, J):
    """ARA_OPT_PRECOMBINED (SURVEY N3 ablation): gathering the tabulated o[e] = FT2(sum_j FT1(l_ej)) gives
    the oracle's YLT and OLT bitwise (integer regime), fixed and ragged trials, and the real regime within
    tolerance of the oracle and bitwise equal to the record path."""
    for integer in (True, False):
        C, elts, layer, yet, N, K = _small_problem(J, integer=integer)
        want = oracle.ylt(C, yet, None, N, K, elts, [layer])
        ctx = _ctx_from(C, elts, [layer])
        ctx.ara_set_option(ara.ARA_OPT_KERNEL, ara.KERNEL_PRESENCE)
        base = gpu_ylt(None, ctx, yet, K=K)
        ctx.ara_set_option(ara.ARA_OPT_PRECOMBINED, 1)
        got = gpu_ylt(None, ctx, yet, K=K)
        assert np.array_equal(got, base), (J, integer)
        if integer:
            assert np.array_equal(got, want), J
            lens = np.random.default_rng(J).integers(0, 200, size=50)
            off = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
            ryet = np.resize(yet, int(off[-1]))
            assert np.array_equal(gpu_ylt(None, ctx, ryet, offsets_np=off),
                                  oracle.ylt(C, ryet, off, len(lens), 0, elts, [layer])), (J, "ragged")
            dev = torch.device("cuda:0")
            ids = torch.from_numpy(yet.view(np.int32)).to(dev)
            ylt = torch.empty((1, N), dtype=torch.float64, device=dev)
            olt = torch.empty((1, N), dtype=torch.float64, device=dev)
            ctx.ara_run_ex(ids, ylt, olt, events_per_trial=K, num_trials=N)
            ctx.ara_check()
            assert np.array_equal(olt.cpu().numpy(), oracle.ylt_olt(C, yet, None, N, K, elts, [layer])[1]), J
        else:
            assert np.all(within_tol(got, want)), J
        ctx.close()


@pytest.mark.parametrize("kw", [dict(inf_limits=True), dict(zero_ret=True), dict(zero_ret=True, inf_limits=True),
                                dict(empty_elts=(0, 2)), dict(integer=False)])
def test_term_edge_cases(cuda_device, kw):
    C, elts, layer, yet, N, K = _small_problem(16, **kw)
    want = oracle.ylt(C, yet, None, N, K, elts, [layer])
    y = gpu_ylt(None, _ctx_from(C, elts, [layer]), yet, K=K)
    if kw.get("integer", True):
        assert np.array_equal(y, want)
    else:
        assert np.all(within_tol(y, want))


def test_ragged_trial_lengths(cuda_device):
    lens = [0, 1, 31, 32, 33, 63, 64, 65, 127, 128, 129, 255, 256, 257, 1000, 1500, 0, 2]
    C, elts, layer, _, _, _ = _small_problem(16)
    rng = np.random.default_rng(5)
    trials = [list(rng.integers(1, C + 1, size=k)) for k in lens]
    ids, off = ragged(trials)
    want = oracle.ylt(C, ids, off, len(trials), 0, elts, [layer])
    ctx = _ctx_from(C, elts, [layer])
    for k, v in variants(ctx):
        assert np.array_equal(gpu_ylt(None, ctx, ids, offsets_np=off, kernel=k, variant=v), want), (k, v)
    # offsets that do not start at 0 (a shard of a bigger YET): prefix junk ids must be ignored
    off2 = off + np.uint64(3)
    ids2 = np.concatenate([np.array([C + 5, 0, 9], np.uint32), ids])
    assert np.array_equal(gpu_ylt(None, ctx, ids2, offsets_np=off2), want)


def test_multi_layer_distinct_widths(cuda_device):
    C, elts, layer, yet, N, K = _small_problem(24, seed=3)
    layers = [layer, ([5, 1, 7], (100.0, 1e6), (0.0, INF)), (list(range(17)), (0.0, INF), (1e5, 2e6)),
              ([23], (0.0, INF), (0.0, INF))]
    want = oracle.ylt(C, yet, None, N, K, elts, layers)
    y = gpu_ylt(None, _ctx_from(C, elts, layers), yet, K=K, num_layers=len(layers))
    assert np.array_equal(y, want)


def test_invalid_ids_reported(cuda_device):
    C, elts, layer, yet, N, K = _small_problem(4)
    ctx = _ctx_from(C, elts, [layer])
    for bad in (0, C + 1, 2**32 - 1):
        y = yet.copy()
        y[17] = bad
        with pytest.raises(ara.AraError) as ei:
            gpu_ylt(None, ctx, y, K=K)
        assert ei.value.status == ara.ARA_E_RANGE
    gpu_ylt(None, ctx, yet, K=K)  # flag was cleared


def test_bad_offsets_reported(cuda_device):
    C, elts, layer, yet, N, K = _small_problem(4)
    ctx = _ctx_from(C, elts, [layer])
    off = np.array([0, 10, 5, 20], np.uint64)
    with pytest.raises(ara.AraError) as ei:
        gpu_ylt(None, ctx, yet[:20], offsets_np=off)
    assert ei.value.status == ara.ARA_E_ARG
    off = np.array([0, 10, 30], np.uint64)
    with pytest.raises(ara.AraError):
        gpu_ylt(None, ctx, yet[:20], offsets_np=off)


def test_determinism_and_launch_shape_invariance_real_regime(cuda_device):
    C, elts, layer, yet, N, K = _small_problem(16, integer=False, N=2000, K=200)
    ctx = _ctx_from(C, elts, [layer])
    base = gpu_ylt(None, ctx, yet, K=K)
    for _ in range(3):
        assert np.array_equal(gpu_ylt(None, ctx, yet, K=K), base)
    for bps in (1, 2, 7):
        ctx.ara_set_option(ara.ARA_OPT_BLOCKS_PER_SM, bps)
        assert np.array_equal(gpu_ylt(None, ctx, yet, K=K), base)
    ctx.ara_set_option(ara.ARA_OPT_BLOCKS_PER_SM, 0)
    for pol in (1, 2, 0):
        ctx.ara_set_option(ara.ARA_OPT_L2_POLICY, pol)
        assert np.array_equal(gpu_ylt(None, ctx, yet, K=K), base)
    for pf in (0, 1):
        ctx.ara_set_option(ara.ARA_OPT_PREFETCH, pf)
        assert ctx.ara_get_option(ara.ARA_OPT_PREFETCH) == pf
        assert np.array_equal(gpu_ylt(None, ctx, yet, K=K), base)
    for k, v in variants(ctx):  # every kernel/variant: same sums up to rounding order
        assert np.all(within_tol(gpu_ylt(None, ctx, yet, K=K, kernel=k, variant=v), base))
    ctx.ara_set_option(ara.ARA_OPT_KERNEL, ara.KERNEL_AUTO)
    assert np.all(within_tol(base, oracle.ylt(C, yet, None, N, K, elts, [layer])))


# ------------------------------------------------------------------ end-to-end host path
def test_run_host_matches_device_path(cuda_device):
    for name in ("T", "V"):
        cfg = synth.Config.load(name)
        elts = synth.make_elts(cfg)
        yet = synth.make_yet(cfg)
        ctx = ara.context_for_config(cfg, elts)
        dev = gpu_ylt(cfg, ctx, yet.event_ids, offsets_np=yet.offsets, K=yet.events_per_trial,
                      num_trials=yet.num_trials)
        ids = torch.from_numpy(yet.event_ids.view(np.int32)).pin_memory()
        out = torch.zeros((1, yet.num_trials), dtype=torch.float64).pin_memory()
        ctx.ara_run_host(ids, out, offsets=yet.offsets, events_per_trial=yet.events_per_trial,
                         num_trials=yet.num_trials)
        assert np.array_equal(out.numpy(), dev)
        pageable = np.zeros((1, yet.num_trials))
        ctx.ara_run_host(yet.event_ids, pageable, offsets=yet.offsets, events_per_trial=yet.events_per_trial,
                         num_trials=yet.num_trials)
        assert np.array_equal(pageable, dev)


# ------------------------------------------------------------------ metrics kernels
@pytest.mark.parametrize("case", ["ties", "uniform", "small", "negzero", "many_rps", "one", "interior_ties",
                                  "dense_bucket", "all_equal", "signed", "two_values", "large"])
def test_metrics_match_oracle(cuda_device, case):
    """metrics_select paths: ranks on the global max/min tie blocks (resolved after the first pass), buckets
    compacted at 16 or 28 bits, interior tie blocks and dense buckets that need every 12-bit pass down to
    the full 64-bit key, negative values, the uncached (n > 8192 per block) path."""
    rng = np.random.default_rng(11)
    rps = [2.0, 5.0, 10.0, 20.0, 25.0, 50.0, 100.0, 200.0, 250.0, 500.0, 1000.0]
    if case == "large":  # > 65,535 keys per block: histograms built in sub-chunks, keys re-read from HBM
        y = np.floor(rng.exponential(1e6, 10_000_019)) * (rng.random(10_000_019) > 0.2)
        rps = [2.0, 10.0, 100.0, 1000.0, 10000.0, 1e6]
    elif case == "interior_ties":  # 40% of the values equal one interior value: the median falls inside it
        y = np.floor(rng.exponential(1e6, 300_000))
        y[rng.random(300_000) < 0.4] = 777_777.0
    elif case == "dense_bucket":  # 200k values within 2^-30 relative of each other (distinct): 64-bit passes
        y = 1e6 + np.arange(200_000, dtype=np.float64) * (1e6 * 2.0 ** -40)
        rng.shuffle(y)
    elif case == "all_equal":
        y = np.full(123_457, 42.5)
    elif case == "signed":  # integer-valued, both signs
        y = np.floor(rng.normal(0.0, 1e5, 400_000))
    elif case == "two_values":
        y = np.where(rng.random(250_000) < 0.5, 3.0, 7.0)
    elif case == "ties":
        y = np.floor(rng.exponential(1000.0, 100_000)) * (rng.random(100_000) > 0.3)
        y[rng.random(100_000) < 0.2] = 4000.0
    elif case == "uniform":
        y = rng.random(1_000_003) * 1e9
    elif case == "small":
        y = np.array([3.0, 1.0, 2.0])
        rps = [1.5, 2.0, 3.0]
    elif case == "negzero":
        y = np.array([0.0, -0.0, 5.0, -0.0, 1.0, 0.0])
        rps = [2.0, 6.0, 1.2]
    elif case == "many_rps":
        y = rng.random(50_000) * 100
        rps = list(np.linspace(1.01, 50_000, 70)) + [8 / 3, 7.0 / 3]
    else:
        y = np.array([42.0])
        rps = []
    if not rps:
        with pytest.raises(ara.AraError):
            ara.ara_pml_tvar(torch.from_numpy(y).cuda(), rps)
        return
    d = torch.from_numpy(y).cuda()
    p, t = ara.ara_pml_tvar(d, rps)
    assert np.array_equal(p, oracle.pml(y, rps))
    assert np.all(within_tol(t, oracle.tvar(y, rps), rel=1e-12, abs_floor=1e-9))
    if case in ("ties", "small", "negzero", "interior_ties", "signed", "two_values", "large"):  # integer-valued: exact
        assert np.array_equal(t, oracle.tvar(y, rps))
    assert np.array_equal(ara.ara_pml(d, rps), p) and np.array_equal(ara.ara_tvar(d, rps), t)
    p2, t2 = ara.ara_pml_tvar(d, rps)
    assert np.array_equal(p2, p) and np.array_equal(t2, t)  # deterministic


# ------------------------------------------------------------------ fake multi-GPU (shards on one GPU)
@pytest.mark.parametrize("name", ["T", "V"])
def test_sharded_runs_reassemble_bitwise(cuda_device, name):
    """Shards run one after another on one GPU (each its own YET buffer, as on G GPUs), reassembled by
    ara_unshard: equal to the oracle over the whole YET (bitwise in the integer regime T, within the
    north_star tolerance in the real regime V) and bitwise to the unsharded GPU run."""
    from paper_1412_4556_b200 import dist
    cfg = synth.Config.load(name)
    elts = synth.make_elts(cfg)
    full = synth.make_yet(cfg)
    want = oracle.ylt_for(cfg, elts, full)
    ctx = ara.context_for_config(cfg, elts)
    single = gpu_ylt(cfg, ctx, full.event_ids, offsets_np=full.offsets, K=full.events_per_trial,
                     num_trials=full.num_trials)
    for G in (2, 3, 8):
        starts = dist.shard_starts(cfg.num_trials, G)
        cap = dist.shard_cap(cfg.num_trials, G)
        gathered = torch.full((G, 1, cap), -1.0, dtype=torch.float64, device=cuda_device)
        for g in range(G):
            y = synth.make_yet(cfg, starts[g], starts[g + 1])
            gathered[g, :, :starts[g + 1] - starts[g]] = torch.from_numpy(
                gpu_ylt(cfg, ctx, y.event_ids, offsets_np=y.offsets, K=y.events_per_trial,
                        num_trials=y.num_trials)).cuda()
        out = torch.empty((1, cfg.num_trials), dtype=torch.float64, device=cuda_device)
        ara.ara_unshard(gathered, G, cap, 1, starts, out)
        torch.cuda.synchronize()
        got = out.cpu().numpy()
        if cfg.regime == "integer":
            assert np.array_equal(got, want), G
        else:
            assert np.all(within_tol(got, want)), G
        assert np.array_equal(got, single), G


# ------------------------------------------------------------------ presence kernel specifics
@pytest.mark.parametrize("C,n,J", [(3_000_000, 20_000, 16),   # bitmap folded mod the shared-memory capacity
                                   (64, 64, 5),                 # every event present: every occurrence hits
                                   (64, 3, 2)])                 # almost nothing present
def test_presence_fold_and_saturation(cuda_device, C, n, J):
    C_, elts, layer, yet, N, K = _small_problem(J, C=C, n=n, N=400, K=301, seed=7)
    want = oracle.ylt(C, yet, None, N, K, elts, [layer])
    ctx = _ctx_from(C, elts, [layer])
    for k, v in variants(ctx):
        assert np.array_equal(gpu_ylt(None, ctx, yet, K=K, kernel=k, variant=v), want), (k, v)


def test_multi_layer_dense_kernel(cuda_device):
    C, elts, layer, yet, N, K = _small_problem(24, seed=4)
    layers = [layer, ([5, 1, 7], (100.0, 1e6), (0.0, INF)), (list(range(17)), (0.0, INF), (1e5, 2e6))]
    want = oracle.ylt(C, yet, None, N, K, elts, layers)
    ctx = _ctx_from(C, elts, layers)
    for k in (ara.KERNEL_DENSE, ara.KERNEL_PRESENCE):
        assert np.array_equal(gpu_ylt(None, ctx, yet, K=K, num_layers=len(layers), kernel=k), want), k


@pytest.mark.parametrize("J", [2, 16, 24, 100])
@pytest.mark.parametrize("C", [1000, 3_000_000, 10_000_000])
def test_trials_with_hit_counts_at_batch_boundaries(cuda_device, J, C):
    """Trials whose number of present events is 0, 1, 31, 32, 33, 64, 96 ... (batch-size multiples),
    in every order; C = 10M also exercises the large-fold (modulo) bitmap path."""
    rng = np.random.default_rng(J * 7 + C % 97)
    present = np.arange(1, 51, dtype=np.uint32)           # events that hold losses
    elts = []
    for j in range(J):
        ids = rng.choice(present, size=rng.integers(1, 51), replace=False).astype(np.uint32)
        elts.append((ids, (rng.integers(1, 1 << 20, size=ids.size)).astype(np.float32),
                     (float(rng.integers(0, 1 << 12)), INF if j % 2 else float(1 << 21))))
    # make every present id hit at least one ELT
    elts[0] = (present, (rng.integers(1, 1 << 20, size=50)).astype(np.float32), (0.0, INF))
    layer = (list(range(J)), (100.0, 1e7), (500.0, 1e9))
    K = 160
    hits = [0, 1, 31, 32, 33, 64, 96, 0, 32, 0, 63, 65, 128, 160, 0]
    trials = []
    for h in hits * 3:
        t = np.concatenate([rng.choice(present, size=h), rng.integers(51, C + 1, size=K - h)]).astype(np.uint32)
        rng.shuffle(t)
        trials.append(t)
    yet = np.concatenate(trials)
    N = len(trials)
    want = oracle.ylt(C, yet, None, N, K, elts, [layer])
    ctx = _ctx_from(C, elts, [layer])
    for k, v in variants(ctx):
        assert np.array_equal(gpu_ylt(None, ctx, yet, K=K, kernel=k, variant=v), want), (k, v)


def test_automatic_kernel_choice(cuda_device):
    """ARA_OPT_KERNEL auto: presence kernel for the paper-shaped layer (sparse bitmap) and for the stress
    layer (10M-event catalogue, 100 ELTs: the folded bitmap sends ~48% of the occurrences to the gather,
    each fetching a 16-B sparse record instead of its 416-B row); dense kernel when most rows hold more
    than two losses and nearly every occurrence would be gathered."""
    rng = np.random.default_rng(3)
    C = 50_000
    dense_elts = [ara.Elt(np.sort(rng.choice(np.arange(1, C + 1, dtype=np.uint32), int(0.9 * C), replace=False)),
                          rng.uniform(1.0, 100.0, int(0.9 * C)).astype(np.float32)) for _ in range(8)]
    ctx = ara.Context(C, dense_elts, [ara.Layer(list(range(8)))])
    st = ctx.ara_layer_stats(0)
    assert st["kernel"] == ara.KERNEL_DENSE and st["est_hit_rate"] > 0.9, st
    ctx.close()
    for name, want in (("T", ara.KERNEL_PRESENCE), ("P", ara.KERNEL_PRESENCE), ("X", ara.KERNEL_PRESENCE)):
        cfg = synth.Config.load(name)
        ctx = ara.context_for_config(cfg, synth.make_elts(cfg))
        st = ctx.ara_layer_stats(0)
        assert st["kernel"] == want, (name, st)
        assert 0 < st["est_hit_rate"] <= 1
        ids = np.unique(np.concatenate([e for e in (synth.make_elts(cfg)[j].event_ids for j in cfg.layers[0].elts)]))
        assert st["present_rows"] == ids.size
        ctx.close()


def test_metrics_fused_and_pass_kernels_agree(cuda_device, monkeypatch):
    """The cooperative fused metric kernel and the 8+1 pass kernels return identical results."""
    rng = np.random.default_rng(21)
    for n in (1, 7, 1000, 300_001, 2_000_000):
        y = np.floor(rng.exponential(1e6, n)) * (rng.random(n) > 0.3)
        y[rng.random(n) < 0.1] = 4e6
        rps = [r for r in synth.return_periods(max(n, 2)) if r <= n] or ([float(n)] if n > 1 else [])
        if not rps:
            continue
        d = torch.from_numpy(y).cuda()
        monkeypatch.delenv("ARA_METRICS_PASSES", raising=False)
        p1, t1 = ara.ara_pml_tvar(d, rps)
        monkeypatch.setenv("ARA_METRICS_PASSES", "1")
        p2, t2 = ara.ara_pml_tvar(d, rps)
        monkeypatch.delenv("ARA_METRICS_PASSES")
        assert np.array_equal(p1, p2) and np.array_equal(p1, oracle.pml(y, rps)), n
        assert np.array_equal(t1, oracle.tvar(y, rps)) and np.array_equal(t2, t1), n


def test_metrics_device_outputs_async(cuda_device):
    """ara_pml_tvar_device: results land in device buffers, enqueued back to back on one stream
    (more than one 16-query batch, and one output omitted), equal to the oracle bitwise."""
    rng = np.random.default_rng(5)
    n = 500_000
    ys = [np.floor(rng.exponential(1e6, n)) * (rng.random(n) > 0.4) for _ in range(3)]
    rps = sorted(set([2.0, 3.0, 5.0, 10.0, 20.0, 25.0, 50.0, 100.0, 200.0, 250.0, 500.0, 1000.0, 2000.0,
                      5000.0, 10000.0, 20000.0, 50000.0, 100000.0, 250000.0, 500000.0, 7.5]))
    assert len(rps) > 16
    s = torch.cuda.Stream()
    ds = [torch.from_numpy(y).cuda() for y in ys]
    torch.cuda.synchronize()
    outs = []
    with torch.cuda.stream(s):
        for i, d in enumerate(ds):
            p = torch.full((len(rps),), -1.0, dtype=torch.float64, device="cuda")
            t = torch.full((len(rps),), -1.0, dtype=torch.float64, device="cuda") if i != 1 else None
            ara.ara_pml_tvar_device(d, rps, p, t, stream=s)
            outs.append((p, t))
    s.synchronize()
    for y, (p, t) in zip(ys, outs):
        assert np.array_equal(p.cpu().numpy(), oracle.pml(y, rps))
        if t is not None:
            assert np.array_equal(t.cpu().numpy(), oracle.tvar(y, rps))
    with pytest.raises(ara.AraError):
        ara.ara_pml_tvar_device(ds[0], [n * 2.0], outs[0][0], None)


def test_metrics_plan_replays_bitwise(cuda_device):
    """ara_metrics_plan_create: a captured PML/TVaR step over three layers (> 16 return periods, strided
    outputs as in a [layers][2][m] result block) equals the oracle bitwise, replay after replay, also after
    the YLT is overwritten between launches (the graph reads the buffer, it caches nothing)."""
    rng = np.random.default_rng(8)
    L, n = 3, 300_000
    rps = [2.0, 5.0, 10.0, 20.0, 25.0, 50.0, 100.0, 200.0, 250.0, 500.0, 1000.0, 2000.0, 5000.0, 10000.0,
           20000.0, 50000.0, 100000.0, 7.5]
    m = len(rps)
    d = torch.empty((L, n), dtype=torch.float64, device="cuda")
    out = torch.full((L, 2, m), -1.0, dtype=torch.float64, device="cuda")
    d.copy_(torch.from_numpy(np.floor(rng.exponential(1e6, (L, n))) * (rng.random((L, n)) > 0.3)))
    plan = ara.ara_metrics_plan_create(d, rps, out[:, 0], out[:, 1], out_stride=2 * m)
    for it in range(3):
        y = np.floor(rng.exponential(1e6 * (it + 1), (L, n))) * (rng.random((L, n)) > 0.3)
        d.copy_(torch.from_numpy(y))
        out.fill_(-1.0)
        plan.launch()
        torch.cuda.synchronize()
        got = out.cpu().numpy()
        for l in range(L):
            assert np.array_equal(got[l, 0], oracle.pml(y[l], rps)), (it, l)
            assert np.array_equal(got[l, 1], oracle.tvar(y[l], rps)), (it, l)
    plan.close()
    with pytest.raises(ara.AraError):
        ara.ara_metrics_plan_create(d, rps, out[:, 0], out[:, 1], out_stride=m - 1)


@pytest.mark.parametrize("layout", [ara.STUDY_INTERLEAVED, ara.STUDY_INDEPENDENT, ara.STUDY_SORTED, ara.STUDY_HASH,
                                    ara.STUDY_INDEX])
def test_section_4b_study_layouts(cuda_device, layout):
    """The Section IV.B data-structure study kernels compute the same YLT."""
    for J, kw in ((16, {}), (3, {}), (24, dict(seed=5))):
        C, elts, layer, yet, N, K = _small_problem(J, **kw)
        want = oracle.ylt(C, yet, None, N, K, elts, [layer])
        ctx = _ctx_from(C, elts, [layer])
        ids = torch.from_numpy(yet.view(np.int32)).cuda()
        out = torch.full((1, N), -1.0, dtype=torch.float64, device=cuda_device)
        ctx.ara_run_study(layout, ids, out, events_per_trial=K, num_trials=N)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), want), (layout, J)
    cfg = synth.Config.load("V")  # variable-length trials, real regime
    elts = synth.make_elts(cfg)
    y = synth.make_yet(cfg, 0, 500)
    want = oracle.ylt_for(cfg, elts, y)
    ctx = ara.context_for_config(cfg, elts)
    out = torch.zeros((1, 500), dtype=torch.float64, device=cuda_device)
    ctx.ara_run_study(layout, torch.from_numpy(y.event_ids.view(np.int32)).cuda(), out,
                      offsets=torch.from_numpy(y.offsets.view(np.int64)).cuda())
    torch.cuda.synchronize()
    assert np.all(within_tol(out.cpu().numpy(), want))


# ------------------------------------------------------------------ N4 outputs
@pytest.mark.parametrize("name", ["T", "V"])
def test_olt_matches_oracle_every_kernel(cuda_device, name):
    cfg = synth.Config.load(name)
    elts = synth.make_elts(cfg)
    yet = synth.make_yet(cfg)
    wy, wo = oracle.ylt_olt(cfg.catalog_size, yet.event_ids, yet.offsets, yet.num_trials, yet.events_per_trial,
                            oracle.config_elts(cfg, elts), oracle.config_layers(cfg))
    ctx = ara.context_for_config(cfg, elts)
    ids = torch.from_numpy(yet.event_ids.view(np.int32)).cuda()
    off = None if yet.offsets is None else torch.from_numpy(yet.offsets.view(np.int64)).cuda()
    for k, v in variants(ctx):
        select(ctx, k, v)
        y = torch.zeros((1, yet.num_trials), dtype=torch.float64, device=cuda_device)
        o = torch.full((1, yet.num_trials), -1.0, dtype=torch.float64, device=cuda_device)
        ctx.ara_run_ex(ids, y, o, offsets=off, events_per_trial=yet.events_per_trial, num_trials=yet.num_trials)
        ctx.ara_check()
        assert np.array_equal(o.cpu().numpy(), wo), (k, v)          # a maximum of identical values: exact
        assert np.all(within_tol(y.cpu().numpy(), wy))
    ctx.ara_set_option(ara.ARA_OPT_KERNEL, ara.KERNEL_AUTO)


def test_olt_wide_rows_and_empty_trials(cuda_device):
    C, elts, layer, _, _, _ = _small_problem(100, seed=9)
    rng = np.random.default_rng(3)
    trials = [list(rng.integers(1, C + 1, size=k)) for k in (0, 1, 5, 40, 0, 100)]
    ids, off = ragged(trials)
    wy, wo = oracle.ylt_olt(C, ids, off, len(trials), 0, elts, [layer])
    ctx = _ctx_from(C, elts, [layer])
    for k, v in variants(ctx):
        select(ctx, k, v)
        y = torch.zeros((1, len(trials)), dtype=torch.float64, device=cuda_device)
        o = torch.full((1, len(trials)), -1.0, dtype=torch.float64, device=cuda_device)
        ctx.ara_run_ex(torch.from_numpy(ids.view(np.int32)).cuda(), y, o,
                       offsets=torch.from_numpy(off.view(np.int64)).cuda())
        assert np.array_equal(o.cpu().numpy(), wo) and np.array_equal(y.cpu().numpy(), wy), (k, v)


def test_aal_ep_and_layer_totals(cuda_device):
    rng = np.random.default_rng(8)
    for n in (1, 1000, 1_000_003):
        y = np.floor(rng.exponential(1e6, n)) * (rng.random(n) > 0.3)
        d = torch.from_numpy(y).cuda()
        assert ara.ara_aal(d) == oracle.aal(y) or abs(ara.ara_aal(d) / oracle.aal(y) - 1) < 1e-12
        xs = [0.0, 1.0, 5e5, 1e6, 3e6, float(y.max()), float(y.max()) + 1]
        assert np.array_equal(ara.ara_ep(d, xs), oracle.ep(y, xs))
    ints = np.floor(rng.exponential(1e6, 100_000))
    assert ara.ara_aal(torch.from_numpy(ints).cuda()) == oracle.aal(ints)  # integer-valued: exact
    cfg = synth.Config.load("T")
    L, n = 5, 777
    ylt = rng.random((L, n)) * 1e6
    group = [0, 1, 0, 2, 1]
    out = torch.zeros((3, n), dtype=torch.float64, device=cuda_device)
    ara.ara_sum_layers(torch.from_numpy(ylt).cuda(), group, 3, out)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), oracle.layer_totals(ylt, group, 3))


# ------------------------------------------------------------------ more edge cases
def test_degenerate_shapes(cuda_device):
    # catalogue of one event; one trial; one ELT; trials made only of that event
    elts = [(np.array([1], np.uint32), np.array([123.0], np.float32), (0.0, INF))]
    layer = ([0], (0.0, INF), (0.0, INF))
    for N, K in ((1, 1), (1, 5), (37, 3)):
        yet = np.ones(N * K, np.uint32)
        want = oracle.ylt(1, yet, None, N, K, elts, [layer])
        ctx = _ctx_from(1, elts, [layer])
        for k, v in variants(ctx):
            assert np.array_equal(gpu_ylt(None, ctx, yet, K=K, num_trials=N, kernel=k, variant=v), want)
    # K = 0: every trial empty
    ctx = _ctx_from(1, elts, [layer])
    y = gpu_ylt(None, ctx, np.zeros(0, np.uint32), K=0, num_trials=4)
    assert np.array_equal(y, np.zeros((1, 4)))


def test_multi_layer_mixed_widths_with_olt_every_kernel(cuda_device):
    C, elts, layer, yet, N, K = _small_problem(40, seed=13)
    layers = [layer, ([3, 1, 7, 9], (10.0, 1e6), (0.0, INF)), (list(range(16)), (0.0, INF), (1e5, 2e6)),
              ([22, 5], (0.0, INF), (0.0, INF)), (list(range(20, 40)), (50.0, 5e5), (0.0, 3e6))]
    wy, wo = oracle.ylt_olt(C, yet, None, N, K, elts, layers)
    ctx = _ctx_from(C, elts, layers)
    ids = torch.from_numpy(yet.view(np.int32)).cuda()
    for k in (ara.KERNEL_AUTO, ara.KERNEL_PRESENCE, ara.KERNEL_DENSE, KERNEL_STREAM):
        select(ctx, k)
        y = torch.zeros((len(layers), N), dtype=torch.float64, device=cuda_device)
        o = torch.zeros((len(layers), N), dtype=torch.float64, device=cuda_device)
        ctx.ara_run_ex(ids, y, o, events_per_trial=K, num_trials=N)
        ctx.ara_check()
        assert np.array_equal(y.cpu().numpy(), wy) and np.array_equal(o.cpu().numpy(), wo), k


def test_host_path_multi_layer_and_unaligned_buffer(cuda_device):
    C, elts, layer, yet, N, K = _small_problem(16, seed=21, N=500, K=99)
    layers = [layer, (list(range(8)), (0.0, INF), (0.0, INF))]
    want = oracle.ylt(C, yet, None, N, K, elts, layers)
    ctx = _ctx_from(C, elts, layers)
    out = np.zeros((2, N))
    ctx.ara_run_host(yet, out, events_per_trial=K, num_trials=N)
    assert np.array_equal(out, want)
    # a device YET starting 4 bytes past an allocation (not 16-B aligned): scalar loads
    padded = torch.from_numpy(np.concatenate([np.zeros(1, np.uint32), yet]).view(np.int32)).cuda()
    y = torch.zeros((2, N), dtype=torch.float64, device=cuda_device)
    ctx.ara_run(padded[1:], y, events_per_trial=K, num_trials=N)
    ctx.ara_check()
    assert np.array_equal(y.cpu().numpy(), want)
