"""Full-size parity at BASELINE.json's paper-shaped configuration (1M trials x 1000 events x 16 ELTs,
2M-event catalogue), in the launch configuration bench.py times (default kernel and variant):

* PI (integer regime): the whole YLT and PML/TVaR bitwise equal to the oracle's (the oracle runs the
  full 1.6e10 lookups on all host cores, ~1 minute);
* P (real regime): 4096 sampled trials within 1e-6 relative / 1e-3 absolute.

The YET is generated on the device by the seeded generator and independently on the host for the
oracle (the two generators are tested bitwise in test_gpu_parity.py)."""
import numpy as np
import pytest
import torch

import oracle
from ara_testutil import within_tol
from paper_1412_4556_b200 import ara, synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _device_run(cfg, elts):
    dev = torch.device("cuda:0")
    n_ids = cfg.num_trials * cfg.kmin
    ids = torch.empty(n_ids, dtype=torch.int32, device=dev)
    synth.yet_ids_device(ids.data_ptr(), cfg.seed, cfg.catalog_size, 0, n_ids, torch.cuda.current_stream().cuda_stream)
    ctx = ara.context_for_config(cfg, elts)
    ylt = torch.empty((len(cfg.layers), cfg.num_trials), dtype=torch.float64, device=dev)
    ctx.ara_run(ids, ylt, events_per_trial=cfg.kmin, num_trials=cfg.num_trials)
    ctx.ara_check()
    rps = synth.return_periods(cfg.num_trials)
    pml, tvar = ara.ara_pml_tvar(ylt[0], rps)
    info = ctx.ara_layer_info(0)
    y = ylt.cpu().numpy()
    del ids
    ctx.close()
    return y, pml, tvar, rps, info


def test_paper_shaped_integer_regime_full_ylt_bitwise(cuda_device):
    cfg = synth.Config.load("PI")
    elts = synth.make_elts(cfg)
    y, pml, tvar, rps, info = _device_run(cfg, elts)
    assert info["variant"].startswith("ara_presence_kernel")
    want = oracle.ylt_for(cfg, elts, synth.make_yet(cfg))
    assert np.array_equal(y, want)
    assert np.array_equal(pml, oracle.pml(want[0], rps))
    assert np.array_equal(tvar, oracle.tvar(want[0], rps))
    assert not np.any(np.signbit(y))


def test_paper_shaped_real_regime_sampled(cuda_device):
    cfg = synth.Config.load("P")
    elts = synth.make_elts(cfg)
    y, pml, tvar, rps, info = _device_run(cfg, elts)
    rng = np.random.default_rng(4556)
    trials = np.unique(np.concatenate([[0, cfg.num_trials - 1], rng.integers(0, cfg.num_trials, 4094)]))
    want = oracle.ylt_for(cfg, elts, synth.make_yet_trials(cfg, trials))
    assert np.all(within_tol(y[0, trials], want[0]))
    # properties of the full YLT that hold at any size
    L3 = cfg.layers[0].agg.limit
    assert np.all(y >= 0) and np.all(y <= L3)
    assert np.all(np.diff(pml) >= 0) and np.all(tvar >= pml)
