"""Shared test helpers (golden fixtures)."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def inf_or(v):
    return float("inf") if v is None else float(v)


def golden_elts(d):
    return [(e["ids"], e["losses"], (e["ft1"][0], inf_or(e["ft1"][1]))) for e in d["elts"]]


def golden_layer(d):
    l = d["layer"]
    return (l["elts"], (l["ft2"][0], inf_or(l["ft2"][1])), (l["ft3"][0], inf_or(l["ft3"][1])))




# ---------------------------------------------------------------- GPU-path helpers (tests only)
def gpu_ylt(cfg_or_none, ctx, event_ids_np, offsets_np=None, K=0, num_trials=None, num_layers=1, variant=None,
            block_threads=None, check=True, kernel=None):
    """Copy a host YET to the device, run ara_run, return the YLT [layers, trials] as numpy."""
    import numpy as np
    import torch
    from paper_1412_4556_b200 import ara
    dev = torch.device("cuda:0")
    ids = torch.from_numpy(np.ascontiguousarray(event_ids_np, dtype=np.uint32).view(np.int32)).to(dev)
    off = None
    if offsets_np is not None:
        off = torch.from_numpy(np.ascontiguousarray(offsets_np, dtype=np.uint64).view(np.int64)).to(dev)
        n = len(offsets_np) - 1
    else:
        n = num_trials if num_trials is not None else (ids.numel() // K if K else 0)
    ylt = torch.full((num_layers, max(n, 1)), -7.0, dtype=torch.float64, device=dev)
    if kernel is not None:
        select(ctx, kernel, variant if variant is not None else 0)
    elif variant is not None:
        ctx.ara_set_option(ara.ARA_OPT_VARIANT, variant)
    if block_threads is not None:
        ctx.ara_set_option(ara.ARA_OPT_BLOCK_THREADS, block_threads)
    ctx.ara_run(ids, ylt, offsets=off, events_per_trial=K, num_trials=n)
    if check:
        ctx.ara_check()
    torch.cuda.synchronize()
    return ylt[:, :n].cpu().numpy()


def golden_context(d, layers_override=None):
    import numpy as np
    from paper_1412_4556_b200 import ara
    elts = [ara.Elt(np.array(e["ids"], np.uint32), np.array(e["losses"], np.float32), e["ft1"][0], inf_or(e["ft1"][1]))
            for e in d["elts"]]
    l = d["layer"]
    layers = layers_override or [ara.Layer(l["elts"], l["ft2"][0], inf_or(l["ft2"][1]), l["ft3"][0], inf_or(l["ft3"][1]))]
    return ara.Context(d["catalog_size"], elts, layers, device=0)


def ragged(trials):
    import numpy as np
    ids = np.array([e for t in trials for e in t], dtype=np.uint32)
    off = np.zeros(len(trials) + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(t) for t in trials])
    return ids, off


def within_tol(gpu, ref, rel=1e-6, abs_floor=1e-3):
    """north_star parity: |gpu - oracle| <= max(1e-6 |oracle|, 1e-3)."""
    import numpy as np
    gpu, ref = np.asarray(gpu), np.asarray(ref)
    return np.abs(gpu - ref) <= np.maximum(rel * np.abs(ref), abs_floor)


KERNEL_STREAM = 2       # test-level selector: the presence path with the fixed-length stream kernel
STREAM_VARIANTS = 10    # ARA_OPT_STREAM = 1..10 (lane 32/24/16; ring; lane XS 24, XS2 24, XS 32/16; mask, mask + L2 prefetch)


def select(ctx, kernel, variant=0):
    """Select a kernel for the next runs: KERNEL_PRESENCE / KERNEL_DENSE variant v with the stream kernel
    off, KERNEL_STREAM = the presence path with stream variant v (it applies to fixed-length YETs with
    K % 4 == 0 and 16-B aligned ids, else the presence kernel runs), KERNEL_AUTO = library defaults."""
    from paper_1412_4556_b200 import ara
    if kernel == KERNEL_STREAM:
        ctx.ara_set_option(ara.ARA_OPT_KERNEL, ara.KERNEL_PRESENCE)
        ctx.ara_set_option(ara.ARA_OPT_STREAM, variant + 1)
        ctx.ara_set_option(ara.ARA_OPT_FILTER, -1)
        return
    ctx.ara_set_option(ara.ARA_OPT_KERNEL, kernel)
    ctx.ara_set_option(ara.ARA_OPT_STREAM, 0)
    ctx.ara_set_option(ara.ARA_OPT_FILTER, -1 if kernel == ara.KERNEL_AUTO else 0)
    if kernel != ara.KERNEL_AUTO:
        ctx.ara_set_option(ara.ARA_OPT_VARIANT, variant)


def variants(ctx):
    """All (kernel, variant) pairs the context can run for its layers' row width (stream variants
    included), leaving the context on the library defaults."""
    from paper_1412_4556_b200 import ara
    out = []
    for k in (ara.KERNEL_PRESENCE, ara.KERNEL_DENSE):
        select(ctx, k, 0)
        out += [(k, v) for v in range(ctx.ara_layer_info(0)["num_variants"])]
    out += [(KERNEL_STREAM, v) for v in range(STREAM_VARIANTS)]
    select(ctx, ara.KERNEL_AUTO)
    return out
