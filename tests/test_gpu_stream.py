"""GPU parity of the fixed-length-trial stream kernel (csrc/stream_kernel.cuh) against the CPU oracle.

The stream kernel is the default ARA path for YETs of fixed-length trials (K % 4 == 0, 16-B aligned ids:
configs P, PI, M, X).  It must give
  * the oracle's YLT BITWISE in the integer regime (every fp64 operation exact), and
    within the north_star tolerance otherwise;
  * the presence kernel's YLT bitwise in every regime (same per-trial summation order), for every
    variant and any trial sharding.
Shapes cover trials much shorter than a batch (K = 4: a batch spans many trials), runs of more than 32
trials without hits (the register ring overflow path), windows with a lane-masked tail (K % 128 != 0),
single-window trials, invalid ids and the occurrence loss table.
"""
import math

import numpy as np
import pytest
import torch

import oracle
from ara_testutil import KERNEL_STREAM, STREAM_VARIANTS, gpu_ylt, select, within_tol
from paper_1412_4556_b200 import ara, synth

pytestmark = pytest.mark.gpu
INF = math.inf
FIXED_KERNELS = ("ara_lane_kernel", "ara_stream_kernel", "ara_mask_kernel")


def _expect_fixed(ctx, v, K):
    """The fixed-length kernel of variant v ran (the mask variants exist for 8 windows per trial only; other
    K fall back to the presence kernel, which must then be the one named)."""
    name = ctx.ara_kernel_name()
    if v in MASK_VARIANTS and (K + 127) // 128 != 8:
        assert name.startswith("ara_presence_kernel"), (v, K, name)
    else:
        assert name.startswith(FIXED_KERNELS), (v, K, name)
LANE_VARIANTS = (0, 1, 2)  # ARA_OPT_STREAM - 1 of the per-lane-queue kernel (32, 24, 16 warps per block)
RING_VARIANT = 3           # the warp-ring kernel


def _problem(J, C, n, K, N, integer=True, seed=0, sparse_yet=False):
    rng = np.random.default_rng(seed + 7919 * J + K)
    elts = []
    for j in range(J):
        ids = rng.choice(np.arange(1, C + 1), size=n, replace=False).astype(np.uint32)
        losses = (rng.integers(1, 1 << 20, size=n) if integer else rng.random(n) * 1e6 + 0.5).astype(np.float32)
        r = float(rng.integers(0, 1 << 18)) if integer else float(rng.integers(0, 1 << 18)) + 0.25
        lim = INF if j % 3 == 1 else float(rng.integers(1 << 18, 1 << 21))
        elts.append((ids, losses, (r, lim)))
    yet = rng.integers(1, C + 1, size=N * K).astype(np.uint32)
    if sparse_yet:  # long runs of trials whose events are absent from every ELT
        present = np.zeros(C + 1, bool)
        for ids, _, _ in elts:
            present[ids] = True
        absent = np.flatnonzero(~present[1:]) + 1
        run = rng.random(N) < 0.85
        for t in np.flatnonzero(run):
            yet[t * K:(t + 1) * K] = rng.choice(absent, size=K)
    layer = (list(range(J)), (5000.0, float(1 << 22)), (2e5, 4e6))
    return elts, layer, yet


def _ctx(C, elts, layers):
    return ara.Context(C, [ara.Elt(i, l, r, lim) for i, l, (r, lim) in elts],
                       [ara.Layer(idx, a[0], a[1], b[0], b[1]) for idx, a, b in layers])


@pytest.mark.parametrize("K", [4, 8, 12, 100, 128, 132, 256, 1000])
def test_stream_bitwise_integer_regime(cuda_device, K):
    C, J = 20_000, 16
    N = max(64, 600_000 // K // 10)
    elts, layer, yet = _problem(J, C, 800, K, N)
    want = oracle.ylt(C, yet, None, N, K, elts, [layer])
    ctx = _ctx(C, elts, [layer])
    for v in range(STREAM_VARIANTS):
        got = gpu_ylt(None, ctx, yet, K=K, num_trials=N, kernel=KERNEL_STREAM, variant=v)
        _expect_fixed(ctx, v, K)
        assert np.array_equal(got, want), (K, v)


@pytest.mark.parametrize("K", [4, 16, 132])
def test_stream_hitless_runs(cuda_device, K):
    """85% of the trials draw only events absent from every ELT: runs far longer than the 32-trial
    register ring, so the kernel must flush and close them (YLT +0) without losing the others."""
    C, J = 50_000, 4
    N = 20_000
    elts, layer, yet = _problem(J, C, 300, K, N, sparse_yet=True)
    want = oracle.ylt(C, yet, None, N, K, elts, [layer])
    assert (want == 0).mean() > 0.8
    ctx = _ctx(C, elts, [layer])
    for v in range(STREAM_VARIANTS):
        assert np.array_equal(gpu_ylt(None, ctx, yet, K=K, num_trials=N, kernel=KERNEL_STREAM, variant=v), want), v


@pytest.mark.parametrize("J", [1, 2, 3, 16, 17, 100, 128])
def test_stream_equals_presence_real_regime(cuda_device, J):
    """Real-valued losses and terms, also for a catalogue larger than the shared bitmap (folded):
    * the warp-ring kernel sums a trial's hits in the presence kernel's order: bitwise equal to it;
    * the per-lane-queue kernel sums by position class: bitwise equal across its variants (the order
      does not depend on the launch shape or the fold) and within tolerance of the presence kernel;
    * all of them within the north_star tolerance of the oracle."""
    for C, n, K, N in ((30_000, 1500, 1000, 3000), (3_000_000, 20_000, 1000, 2000)):
        elts, layer, yet = _problem(J, C, n, K, N, integer=False, seed=5)
        want = oracle.ylt(C, yet, None, N, K, elts, [layer])
        ctx = _ctx(C, elts, [layer])
        pres = gpu_ylt(None, ctx, yet, K=K, num_trials=N, kernel=ara.KERNEL_PRESENCE, variant=0)
        assert ctx.ara_kernel_name().startswith("ara_presence_kernel")
        ring = gpu_ylt(None, ctx, yet, K=K, num_trials=N, kernel=KERNEL_STREAM, variant=RING_VARIANT)
        assert ctx.ara_kernel_name().startswith("ara_stream_kernel")
        assert np.array_equal(ring, pres), (J, C)
        lanes = [gpu_ylt(None, ctx, yet, K=K, num_trials=N, kernel=KERNEL_STREAM, variant=v) for v in LANE_VARIANTS]
        assert ctx.ara_kernel_name().startswith("ara_lane_kernel")
        for y in lanes[1:]:
            assert np.array_equal(y, lanes[0]), (J, C)
        assert np.all(within_tol(lanes[0], pres)), (J, C)
        assert np.all(within_tol(pres, want)) and np.all(within_tol(lanes[0], want)), (J, C)


def test_stream_sharding_invariant_and_vs_oracle(cuda_device):
    """Trial blocks of a sharded run (each shard its own YET buffer, as on G GPUs) reassemble to the
    unsharded YLT bitwise, and both equal the oracle within tolerance (real regime)."""
    cfg = synth.Config.load("P")
    elts = synth.make_elts(cfg)
    N, K = 12_000, cfg.kmin
    ids = synth.yet_ids(cfg.seed, cfg.catalog_size, 0, N * K)
    ctx = ara.context_for_config(cfg, elts)
    select(ctx, KERNEL_STREAM, 0)
    whole = gpu_ylt(None, ctx, ids, K=K, num_trials=N)
    assert ctx.ara_kernel_name().startswith("ara_lane_kernel")
    for G in (2, 3, 8):
        starts = [(g * N) // G for g in range(G + 1)]
        parts = [gpu_ylt(None, ctx, ids[starts[g] * K:starts[g + 1] * K], K=K, num_trials=starts[g + 1] - starts[g])
                 for g in range(G)]
        assert np.array_equal(np.concatenate(parts, axis=1), whole), G
    sample = np.arange(0, N, 7)
    want = oracle.ylt_for(cfg, elts, synth.make_yet_trials(cfg, sample))
    assert np.all(within_tol(whole[:, sample], want))


def test_stream_olt_and_invalid_ids(cuda_device):
    C, J, K, N = 20_000, 16, 1000, 500
    elts, layer, yet = _problem(J, C, 800, K, N, seed=3)
    wy, wo = oracle.ylt_olt(C, yet, None, N, K, elts, [layer])
    ctx = _ctx(C, elts, [layer])
    ids = torch.from_numpy(yet.view(np.int32)).cuda()
    for v in range(STREAM_VARIANTS):
        select(ctx, KERNEL_STREAM, v)
        y = torch.zeros((1, N), dtype=torch.float64, device=cuda_device)
        o = torch.full((1, N), -1.0, dtype=torch.float64, device=cuda_device)
        ctx.ara_run_ex(ids, y, o, events_per_trial=K, num_trials=N)
        ctx.ara_check()
        _expect_fixed(ctx, v, K)
        assert np.array_equal(y.cpu().numpy(), wy) and np.array_equal(o.cpu().numpy(), wo), v
    for bad in (0, C + 1, 2**32 - 1):
        b = yet.copy()
        b[K * 123 + 17] = bad
        select(ctx, KERNEL_STREAM, 0)
        with pytest.raises(ara.AraError) as e:
            gpu_ylt(None, ctx, b, K=K, num_trials=N)
        assert e.value.status == ara.ARA_E_RANGE
        # a valid run afterwards is clean again
        assert np.array_equal(gpu_ylt(None, ctx, yet, K=K, num_trials=N), wy)


def test_plan_replays_eager_step_bitwise(cuda_device):
    """ara_plan: the captured step (ara_run + PML/TVaR of every layer) replayed as a CUDA graph gives the
    eager calls' YLT and metrics bit for bit, replay after replay; multi-layer, fixed-length YET."""
    C, J, K, N = 20_000, 16, 1000, 3000
    elts, layer, yet = _problem(J, C, 800, K, N, integer=False, seed=11)
    layers = [layer, (list(range(8)), (100.0, 5e6), (1e4, 3e6))]
    ctx = _ctx(C, elts, layers)
    ids = torch.from_numpy(yet.view(np.int32)).cuda()
    rps = synth.return_periods(N)
    m = len(rps)
    y_e = torch.zeros((2, N), dtype=torch.float64, device=cuda_device)
    ctx.ara_run(ids, y_e, events_per_trial=K, num_trials=N)
    ctx.ara_check()
    want_p = [ara.ara_pml_tvar(y_e[l], rps) for l in range(2)]
    y = torch.full((2, N), -1.0, dtype=torch.float64, device=cuda_device)
    pml = torch.zeros((2, m), dtype=torch.float64, device=cuda_device)
    tvar = torch.zeros((2, m), dtype=torch.float64, device=cuda_device)
    plan = ctx.ara_plan_create(ids, y, rps, pml, tvar, events_per_trial=K, num_trials=N)
    for _ in range(3):
        y.fill_(-1.0)
        pml.zero_()
        plan.launch()
        torch.cuda.synchronize()
        assert torch.equal(y, y_e)
        for l in range(2):
            assert np.array_equal(pml[l].cpu().numpy(), want_p[l][0]) and np.array_equal(tvar[l].cpu().numpy(), want_p[l][1])
    ctx.ara_check()
    want = oracle.ylt(C, yet, None, N, K, elts, layers)
    assert np.all(within_tol(y.cpu().numpy(), want))
    plan.close()


def _sparse_problem(J, C, n, K, N, seed, integer=True):
    """ELTs of n distinct ids each over a large catalogue (drawn without materialising it)."""
    rng = np.random.default_rng(seed)
    elts = []
    for j in range(J):
        ids = np.unique(rng.integers(1, C + 1, size=2 * n))[:n]
        rng.shuffle(ids)
        losses = (rng.integers(1, 1 << 20, size=ids.size) if integer else rng.random(ids.size) * 1e6 + 0.5)
        elts.append((ids.astype(np.uint32), losses.astype(np.float32),
                     (float(rng.integers(0, 1 << 16)), INF if j % 3 == 1 else float(rng.integers(1 << 18, 1 << 21)))))
    yet = rng.integers(1, C + 1, size=N * K).astype(np.uint32)
    layer = (list(range(J)), (5000.0, float(1 << 24)), (2e5, 4e7))
    return elts, layer, yet


def test_exact_scan_filter_stress_shape(cuda_device):
    """Config X's shape (J = 100 ELTs of 10,000 entries over a 10M-event catalogue: the shared bitmap is
    folded ~6.6x, ~48% of occurrences are candidates, ~80% of them false positives).  The lane kernel
    with the exact scan filter (chosen automatically) equals the oracle bitwise (integer regime) for
    every XS variant, also with the occurrence loss table, and the plain lane / presence kernels."""
    C, J, n, K, N = 10_000_000, 100, 10_000, 1000, 1500
    elts, layer, yet = _sparse_problem(J, C, n, K, N, seed=17)
    wy, wo = oracle.ylt_olt(C, yet, None, N, K, elts, [layer])
    ctx = _ctx(C, elts, [layer])
    select(ctx, ara.KERNEL_AUTO)
    got = gpu_ylt(None, ctx, yet, K=K, num_trials=N)
    assert ",XS" in ctx.ara_kernel_name(), ctx.ara_kernel_name()
    assert np.array_equal(got, wy)
    for v in (4, 5, 6, 7, 0):  # XS 24, XS2 24, XS 32/16 warps, plain lane kernel
        assert np.array_equal(gpu_ylt(None, ctx, yet, K=K, num_trials=N, kernel=KERNEL_STREAM, variant=v), wy), v
    assert np.array_equal(gpu_ylt(None, ctx, yet, K=K, num_trials=N, kernel=ara.KERNEL_PRESENCE, variant=0), wy)
    select(ctx, ara.KERNEL_AUTO)
    ids = torch.from_numpy(yet.view(np.int32)).cuda()
    y = torch.zeros((1, N), dtype=torch.float64, device=cuda_device)
    o = torch.full((1, N), -1.0, dtype=torch.float64, device=cuda_device)
    ctx.ara_run_ex(ids, y, o, events_per_trial=K, num_trials=N)
    ctx.ara_check()
    assert np.array_equal(y.cpu().numpy(), wy) and np.array_equal(o.cpu().numpy(), wo)
    # invalid ids are still reported through the exact filter
    b = yet.copy()
    b[K * 7 + 3] = C + 5
    with pytest.raises(ara.AraError):
        gpu_ylt(None, ctx, b, K=K, num_trials=N)


def test_exact_scan_filter_compact_records_dense(cuda_device):
    """The exact scan filter's compact-row index (rank over the unfolded bitmap, records of the
    loss-holding rows only) on a small, dense catalogue: rows with 1..8 losses (rows with > 2 read in
    full via the record's event id), loss-holding rows at every position of a bitmap word (ids 31, 32,
    63, 64, ...), the last row C, and invalid ids reported.  Every XS variant equals the oracle bitwise
    (integer regime) and the plain lane kernel."""
    C, J, K, N = 4099, 8, 256, 600
    rng = np.random.default_rng(23)
    elts = []
    for j in range(J):
        ids = np.unique(np.concatenate([rng.integers(1, C + 1, size=900), [31, 32, 63, 64, 1, C]]))
        rng.shuffle(ids)
        losses = rng.integers(1, 1 << 20, size=ids.size)
        elts.append((ids.astype(np.uint32), losses.astype(np.float32), (float(rng.integers(0, 1 << 12)), float(1 << 21))))
    layer = (list(range(J)), (3000.0, float(1 << 24)), (1e5, 4e7))
    yet = rng.integers(1, C + 1, size=N * K).astype(np.uint32)
    yet[:8] = [31, 32, 63, 64, 1, C, 33, 62]
    want = oracle.ylt(C, yet, None, N, K, elts, [layer])
    ctx = _ctx(C, elts, [layer])
    for v in (4, 5, 6, 7):  # XS 24, XS2 24, XS 32/16 warps
        got = gpu_ylt(None, ctx, yet, K=K, num_trials=N, kernel=KERNEL_STREAM, variant=v)
        assert ",XS" in ctx.ara_kernel_name(), ctx.ara_kernel_name()
        assert np.array_equal(got, want), v
    assert np.array_equal(gpu_ylt(None, ctx, yet, K=K, num_trials=N, kernel=KERNEL_STREAM, variant=0), want)
    for bad in (C + 1, 0, 0xFFFFFFFF):
        b = yet.copy()
        b[K * 5 + 77] = bad
        with pytest.raises(ara.AraError):
            gpu_ylt(None, ctx, b, K=K, num_trials=N, kernel=KERNEL_STREAM, variant=4)
    ctx.close()


def test_exact_scan_filter_full_queues(cuda_device):
    """Every id of the catalogue holds a loss (each lane queues a hit for every slot of every window): the
    lane queues run full at every trial end, where the two-window deferral (XS2) flushes two pending windows
    (8 entries per lane) -- the queue must be drained between them.  Every XS variant equals the oracle
    bitwise (integer regime)."""
    C, J, K, N = 2048, 4, 1000, 700
    rng = np.random.default_rng(29)
    elts = []
    for j in range(J):
        ids = np.arange(1, C + 1, dtype=np.uint32) if j == 0 else np.unique(rng.integers(1, C + 1, size=700)).astype(np.uint32)
        rng.shuffle(ids)
        elts.append((ids, rng.integers(1, 1 << 20, size=ids.size).astype(np.float32), (float(rng.integers(0, 1 << 12)), float(1 << 21))))
    layer = (list(range(J)), (3000.0, float(1 << 24)), (1e5, 4e9))
    yet = rng.integers(1, C + 1, size=N * K).astype(np.uint32)
    want = oracle.ylt(C, yet, None, N, K, elts, [layer])
    ctx = _ctx(C, elts, [layer])
    ctx.ara_set_option(ara.ARA_OPT_FILTER, 1)
    for v in (4, 5, 6, 7):  # XS 24, XS2 24, XS 32/16 warps
        ctx.ara_set_option(ara.ARA_OPT_KERNEL, ara.KERNEL_PRESENCE)
        ctx.ara_set_option(ara.ARA_OPT_STREAM, v + 1)
        got = gpu_ylt(None, ctx, yet, K=K, num_trials=N)
        assert ",XS" in ctx.ara_kernel_name(), ctx.ara_kernel_name()
        assert np.array_equal(got, want), v
    ctx.close()


def test_exact_scan_filter_config_x_sampled(cuda_device):
    """Config X itself (real regime) on a 20,000-trial slice generated on the device: the automatic
    kernel (lane + exact scan filter) within tolerance of the oracle on 500 sampled trials and of the
    presence kernel on every trial."""
    cfg = synth.Config.load("X")
    elts = synth.make_elts(cfg)
    N, K = 20_000, cfg.kmin
    ids = torch.empty(N * K, dtype=torch.int32, device=cuda_device)
    synth.yet_ids_device(ids.data_ptr(), cfg.seed, cfg.catalog_size, 0, N * K, torch.cuda.current_stream().cuda_stream)
    ctx = ara.context_for_config(cfg, elts)
    y = torch.zeros((1, N), dtype=torch.float64, device=cuda_device)
    ctx.ara_run(ids, y, events_per_trial=K, num_trials=N)
    ctx.ara_check()
    assert ",XS" in ctx.ara_kernel_name(), ctx.ara_kernel_name()
    got = y.cpu().numpy()
    select(ctx, ara.KERNEL_PRESENCE, 0)
    ctx.ara_run(ids, y, events_per_trial=K, num_trials=N)
    ctx.ara_check()
    # two summation orders: they agree to rounding, which FT3's subtraction of the retention can amplify
    # (S_n close to R3); the bar between kernels is the north_star tolerance
    assert np.all(within_tol(got, y.cpu().numpy()))
    sample = np.arange(0, N, 40)
    want = oracle.ylt_for(cfg, elts, synth.make_yet_trials(cfg, sample))
    assert np.all(within_tol(got[:, sample], want))


@pytest.mark.parametrize("name", ["P", "X"])
def test_variant_groups_bitwise_real_regime(cuda_device, name):
    """Every kernel family on a 20,000-trial slice of a real-regime configuration (device-generated YET):
    kernels that share a summation order agree BIT FOR BIT -- {presence, warp ring}, {every lane-queue and
    exact-filter variant}, {the two mask variants} -- and every family is within the north_star tolerance
    of the oracle on sampled trials.  (A lost hit in one variant showed up only here: integer-regime tests
    on small shapes had passed.)"""
    cfg = synth.Config.load(name)
    elts = synth.make_elts(cfg)
    N, K = 20_000, cfg.kmin
    ids = torch.empty(N * K, dtype=torch.int32, device=cuda_device)
    synth.yet_ids_device(ids.data_ptr(), cfg.seed, cfg.catalog_size, 0, N * K, torch.cuda.current_stream().cuda_stream)
    ctx = ara.context_for_config(cfg, elts)

    def run(kernel, v=0):
        select(ctx, kernel, v)
        y = torch.full((1, N), -1.0, dtype=torch.float64, device=cuda_device)
        ctx.ara_run(ids, y, events_per_trial=K, num_trials=N)
        ctx.ara_check()
        return ctx.ara_kernel_name(), y.cpu().numpy()

    groups = {"presence": [run(ara.KERNEL_PRESENCE, 0), run(KERNEL_STREAM, RING_VARIANT)],
              "lane": [run(KERNEL_STREAM, v) for v in LANE_VARIANTS + (4, 5, 6, 7)],
              "mask": [run(KERNEL_STREAM, v) for v in MASK_VARIANTS]}
    sample = np.arange(0, N, 100)
    want = oracle.ylt_for(cfg, elts, synth.make_yet_trials(cfg, sample))
    for g, runs in groups.items():
        first_name, first = runs[0]
        for kname, y in runs[1:]:
            assert np.array_equal(y, first), (g, first_name, kname, int((y != first).sum()))
        assert np.all(within_tol(first[:, sample], want)), g
        assert np.all(within_tol(first, groups["presence"][0][1])), g
    ctx.close()


# ------------------------------------------------------------------ fused multi-layer pass
def _layers_distinct(J_list, C, seed, integer=True, shared=False, n=800):
    """Layers over distinct ELTs (config M's reading c20), or all over the same ELTs (`shared`, the tower)."""
    rng = np.random.default_rng(seed)
    elts, layers, e0 = [], [], 0
    for li, J in enumerate(J_list):
        if not shared or li == 0:
            for j in range(J):
                ids = rng.choice(np.arange(1, C + 1), size=n, replace=False).astype(np.uint32)
                losses = (rng.integers(1, 1 << 20, size=n) if integer else rng.random(n) * 1e6 + 0.5).astype(np.float32)
                r = float(rng.integers(0, 1 << 16)) + (0.0 if integer else 0.25)
                elts.append((ids, losses, (r, INF if j % 3 == 1 else float(rng.integers(1 << 18, 1 << 21)))))
        idx = list(range(J)) if shared else list(range(e0, e0 + J))
        e0 += 0 if shared else J
        layers.append((idx, (float(1000 * li), float((li + 2) << 21)), (float(5e4 * li), 4e6 + 1e6 * li)))
    return elts, layers


@pytest.mark.parametrize("J_list,shared", [([16] * 8, False), ([3, 16, 1, 40, 7], False), ([16] * 20, False),
                                           ([16] * 4, True)])
def test_fused_layers_bitwise(cuda_device, J_list, shared):
    """One pass for several layers: integer regime bitwise vs the oracle (distinct ELTs as config M; mixed
    widths; 20 layers = two fused groups; a tower of layers sharing ELTs, whose events hold > 4 entries and
    take the full-row path), and bitwise equal to layer-outer runs of the single-layer lane kernel in the
    real regime (the same per-layer summation order)."""
    C, K, N = 20_000, 1000, 1200
    elts, layers = _layers_distinct(J_list, C, seed=len(J_list) + 7 * shared)
    rng = np.random.default_rng(5)
    yet = rng.integers(1, C + 1, size=N * K).astype(np.uint32)
    want = oracle.ylt(C, yet, None, N, K, elts, layers)
    ctx = _ctx(C, elts, layers)
    select(ctx, ara.KERNEL_AUTO)
    ctx.ara_set_option(ara.ARA_OPT_FUSED, 1)
    got = gpu_ylt(None, ctx, yet, K=K, num_trials=N, num_layers=len(layers))
    assert ctx.ara_kernel_name().startswith("ara_fused_kernel"), ctx.ara_kernel_name()
    assert np.array_equal(got, want)
    ctx.ara_set_option(ara.ARA_OPT_FUSED, 0)
    assert np.array_equal(gpu_ylt(None, ctx, yet, K=K, num_trials=N, num_layers=len(layers)), want)
    ctx.close()
    # real regime: fused == layer-outer lane kernel, bit for bit
    elts, layers = _layers_distinct(J_list, C, seed=3, integer=False, shared=shared)
    ctx = _ctx(C, elts, layers)
    select(ctx, ara.KERNEL_AUTO)
    ctx.ara_set_option(ara.ARA_OPT_FUSED, 1)
    fused = gpu_ylt(None, ctx, yet, K=K, num_trials=N, num_layers=len(layers))
    assert ctx.ara_kernel_name().startswith("ara_fused_kernel")
    select(ctx, KERNEL_STREAM, 0)
    outer = gpu_ylt(None, ctx, yet, K=K, num_trials=N, num_layers=len(layers))
    assert ctx.ara_kernel_name().startswith("ara_lane_kernel")
    assert np.array_equal(fused, outer)
    assert np.all(within_tol(fused, oracle.ylt(C, yet, None, N, K, elts, layers)))


def test_fused_config_m_sampled(cuda_device):
    """Config M (8 layers x 16 distinct ELTs, real regime) on 30,000 device-generated trials: the fused
    pass within tolerance of the oracle on sampled trials and of the layer-outer presence kernel
    everywhere."""
    cfg = synth.Config.load("M")
    elts = synth.make_elts(cfg)
    N, K, L = 30_000, cfg.kmin, len(cfg.layers)
    ids = torch.empty(N * K, dtype=torch.int32, device=cuda_device)
    synth.yet_ids_device(ids.data_ptr(), cfg.seed, cfg.catalog_size, 0, N * K, torch.cuda.current_stream().cuda_stream)
    ctx = ara.context_for_config(cfg, elts)
    ctx.ara_set_option(ara.ARA_OPT_FUSED, 1)
    y = torch.zeros((L, N), dtype=torch.float64, device=cuda_device)
    ctx.ara_run(ids, y, events_per_trial=K, num_trials=N)
    ctx.ara_check()
    assert ctx.ara_kernel_name().startswith("ara_fused_kernel")
    fused = y.cpu().numpy()
    ctx.ara_set_option(ara.ARA_OPT_FUSED, 0)
    ctx.ara_run(ids, y, events_per_trial=K, num_trials=N)
    ctx.ara_check()
    assert np.all(within_tol(fused, y.cpu().numpy()))
    sample = np.arange(0, N, 60)
    want = oracle.ylt_for(cfg, elts, synth.make_yet_trials(cfg, sample))
    assert np.all(within_tol(fused[:, sample], want))


# ------------------------------------------------------------------ candidate-mask kernel
MASK_VARIANTS = (8, 9)  # ARA_OPT_STREAM - 1: mask kernel without / with the per-lane L2 prefetch


@pytest.mark.parametrize("K", [900, 1000, 1024])  # the mask kernel is built for 8 windows per trial
def test_mask_kernel_bitwise(cuda_device, K):
    """The candidate-mask kernel (trials of <= 1024 occurrences): integer regime bitwise vs the oracle for
    every variant, incl. trials with more candidates than one staging chunk (dense layer), OLT, and its
    fixed order (bitwise equal across launch shapes)."""
    C, J = 20_000, 16
    N = max(64, 600_000 // K // 10)
    for n in (800, 8000):  # 8000 entries per ELT: ~100% of the rows present, > 256 candidates per trial
        elts, layer, yet = _problem(J, C, n, K, N)
        wy, wo = oracle.ylt_olt(C, yet, None, N, K, elts, [layer])
        ctx = _ctx(C, elts, [layer])
        for v in MASK_VARIANTS:
            got = gpu_ylt(None, ctx, yet, K=K, num_trials=N, kernel=KERNEL_STREAM, variant=v)
            assert ctx.ara_kernel_name().startswith("ara_mask_kernel"), ctx.ara_kernel_name()
            assert np.array_equal(got, wy), (K, n, v)
        select(ctx, KERNEL_STREAM, MASK_VARIANTS[0])
        ids = torch.from_numpy(yet.view(np.int32)).cuda()
        y = torch.zeros((1, N), dtype=torch.float64, device=cuda_device)
        o = torch.full((1, N), -1.0, dtype=torch.float64, device=cuda_device)
        ctx.ara_run_ex(ids, y, o, events_per_trial=K, num_trials=N)
        ctx.ara_check()
        assert np.array_equal(y.cpu().numpy(), wy) and np.array_equal(o.cpu().numpy(), wo), (K, n)


def test_mask_kernel_real_regime_and_invalid_ids(cuda_device):
    C, J, K, N = 3_000_000, 16, 1000, 2000
    elts, layer, yet = _problem(J, C, 20_000, K, N, integer=False, seed=5)
    want = oracle.ylt(C, yet, None, N, K, elts, [layer])
    ctx = _ctx(C, elts, [layer])
    ys = [gpu_ylt(None, ctx, yet, K=K, num_trials=N, kernel=KERNEL_STREAM, variant=v) for v in MASK_VARIANTS]
    assert np.array_equal(ys[0], ys[1])
    assert np.all(within_tol(ys[0], want))
    select(ctx, KERNEL_STREAM, MASK_VARIANTS[0])
    for bad in (0, C + 1, 2**32 - 1):
        b = yet.copy()
        b[K * 77 + 5] = bad
        with pytest.raises(ara.AraError) as e:
            gpu_ylt(None, ctx, b, K=K, num_trials=N)
        assert e.value.status == ara.ARA_E_RANGE
    assert np.array_equal(gpu_ylt(None, ctx, yet, K=K, num_trials=N), ys[0])
