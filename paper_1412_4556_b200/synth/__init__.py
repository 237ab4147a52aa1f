"""Seeded synthetic ARA inputs ("ARA-GEN-1"): the ONE module both the CUDA path and the oracle may use.

It holds none of the method's arithmetic (no lookup, no financial terms, no sums): only a
counter-based integer PRNG and the recipe that turns its draws into a YET and ELTs of the
paper's shapes.  The paper gives shapes only -- 1M trials x 1000 events, 16 ELTs of
"tens of thousands" of entries (Section III/IV.C); the value
distributions are this build's.

Generator:
    sm64(x)       SplitMix64 finaliser of x + 0x9E3779B97F4A7C15
    key(s)        sm64(seed ^ s * 0xD1B54A32D192ED03)
    draw(s, i)    sm64(key(s) + i)                  -- counter based: any index, any order
    uni(r, n)     ((r >> 32) * n) >> 32             -- n < 2**32
Streams s = kind * 2**32 + g:  kind 1 YET ids, 2 trial lengths, 3 ELT ids, 4 ELT losses,
5 ELT loss fractions (real regime); g = ELT index.

YET id of global occurrence q:  1 + uni(draw(S_YET, q), C).  Ids are i.i.d. uniform over the
catalogue, so storage order is a valid time order.  The device generator
(`synth.cu`, ``ara_synth_yet_ids``) implements the same integer recipe and is tested bitwise
against :func:`yet_ids` here.

Integer regime loss:  (1 + (r >> 44)) << popcount(r & 0xFF), an integer in [1, 2**28], exact in
fp32.  Real regime:  fp32_RN(loss_int * (1 + u/3)),  u = (r' >> 40) / 2**24, evaluated in double.
"""
from __future__ import annotations

import ctypes
import json
import math
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

SEED = 14124556  # the arXiv id

_M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB
STREAM_MUL = 0xD1B54A32D192ED03

KIND_YET_IDS = 1
KIND_TRIAL_LEN = 2
KIND_ELT_IDS = 3
KIND_ELT_LOSS = 4
KIND_ELT_FRAC = 5


def stream(kind: int, g: int = 0) -> int:
    return ((kind << 32) + g) & _M64


# ---------------------------------------------------------------- scalar (pure Python) reference
def sm64_int(x: int) -> int:
    x = (x + GOLDEN) & _M64
    z = x
    z = ((z ^ (z >> 30)) * MIX1) & _M64
    z = ((z ^ (z >> 27)) * MIX2) & _M64
    return z ^ (z >> 31)


def key_int(seed: int, s: int) -> int:
    return sm64_int((seed ^ ((s * STREAM_MUL) & _M64)) & _M64)


def draw_int(seed: int, s: int, i: int) -> int:
    return sm64_int((key_int(seed, s) + i) & _M64)


def uni_int(r: int, n: int) -> int:
    return ((r >> 32) * n) >> 32


# ---------------------------------------------------------------- vectorised numpy
def _sm64_np(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = x + np.uint64(GOLDEN)
        z = (x ^ (x >> np.uint64(30))) * np.uint64(MIX1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(MIX2)
        return z ^ (z >> np.uint64(31))


def draws(seed: int, s: int, start: int, count: int) -> np.ndarray:
    """draw(s, i) for i in [start, start+count) as uint64."""
    k = np.uint64(key_int(seed, s))
    i = np.arange(count, dtype=np.uint64) + np.uint64(start)
    with np.errstate(over="ignore"):
        return _sm64_np(i + k)


def draws_at(seed: int, s: int, idx: np.ndarray) -> np.ndarray:
    k = np.uint64(key_int(seed, s))
    with np.errstate(over="ignore"):
        return _sm64_np(np.asarray(idx, dtype=np.uint64) + k)


def uni_np(r: np.ndarray, n: int) -> np.ndarray:
    return ((r >> np.uint64(32)) * np.uint64(n)) >> np.uint64(32)


# ---------------------------------------------------------------- YET
def yet_ids(seed: int, catalog_size: int, q0: int, count: int) -> np.ndarray:
    """Event ids of global occurrences q0 .. q0+count-1 (uint32, values in [1, C])."""
    if not (1 <= catalog_size < 2**32):
        raise ValueError("catalog_size must be in [1, 2**32)")
    r = draws(seed, stream(KIND_YET_IDS), q0, count)
    return (uni_np(r, catalog_size) + np.uint64(1)).astype(np.uint32)


def yet_ids_chunked(seed: int, catalog_size: int, q0: int, count: int, chunk: int = 1 << 26) -> np.ndarray:
    """Same as yet_ids, generated in chunks (bounded host memory for multi-GB YETs)."""
    out = np.empty(count, dtype=np.uint32)
    for a in range(0, count, chunk):
        b = min(count, a + chunk)
        out[a:b] = yet_ids(seed, catalog_size, q0 + a, b - a)
    return out


def trial_lengths(seed: int, t0: int, count: int, kmin: int, kmax: int) -> np.ndarray:
    if kmin == kmax:
        return np.full(count, kmin, dtype=np.uint64)
    r = draws(seed, stream(KIND_TRIAL_LEN), t0, count)
    return uni_np(r, kmax - kmin + 1) + np.uint64(kmin)


def trial_offsets(seed: int, num_trials: int, kmin: int, kmax: int) -> np.ndarray:
    """Exclusive prefix sum of trial lengths, length N+1 (uint64)."""
    lens = trial_lengths(seed, 0, num_trials, kmin, kmax)
    off = np.zeros(num_trials + 1, dtype=np.uint64)
    np.cumsum(lens, out=off[1:])
    return off


# ---------------------------------------------------------------- ELTs
def elt_event_ids(seed: int, g: int, n: int, catalog_size: int) -> np.ndarray:
    """First n distinct ids of the stream 1 + uni(draw(3*2^32+g, i), C), in draw order."""
    if n > catalog_size:
        raise ValueError("ELT entry count exceeds the catalogue")
    s = stream(KIND_ELT_IDS, g)
    got = np.empty(0, dtype=np.uint64)
    start = 0
    batch = max(1024, 2 * n)
    while True:
        ids = uni_np(draws(seed, s, start, batch), catalog_size) + np.uint64(1)
        allids = np.concatenate([got, ids]) if got.size else ids
        # keep first occurrences in draw order
        _, first = np.unique(allids, return_index=True)
        first.sort()
        uniq = allids[first]
        if uniq.size >= n:
            return uniq[:n].astype(np.uint32)
        got = allids
        start += batch
        batch *= 2


def elt_losses(seed: int, g: int, n: int, regime: str = "integer") -> np.ndarray:
    """fp32 losses, strictly positive and finite."""
    r = draws(seed, stream(KIND_ELT_LOSS, g), 0, n)
    base = (np.uint64(1) + (r >> np.uint64(44)))
    pc = _popcount8(r & np.uint64(0xFF))
    loss_int = base << pc  # <= 2**28, exact in fp32 and fp64
    if regime == "integer":
        return loss_int.astype(np.float32)
    if regime != "real":
        raise ValueError(regime)
    r2 = draws(seed, stream(KIND_ELT_FRAC, g), 0, n)
    u = (r2 >> np.uint64(40)).astype(np.float64) / float(1 << 24)
    t = 1.0 + u / 3.0
    return (loss_int.astype(np.float64) * t).astype(np.float32)


def _popcount8(x: np.ndarray) -> np.ndarray:
    c = np.zeros_like(x)
    for b in range(8):
        c += (x >> np.uint64(b)) & np.uint64(1)
    return c


def loss_mean_integer() -> float:
    """Closed-form mean of the integer-regime loss: E[1+U20] * E[2^Bin(8,1/2)] = (2^20+1)/2 * 1.5^8."""
    return (2**20 + 1) / 2.0 * 1.5**8


# ---------------------------------------------------------------- configs
@dataclass
class Terms:
    retention: float
    limit: float  # may be +inf

    @staticmethod
    def from_json(v) -> "Terms":
        r, l = v
        return Terms(float(r), math.inf if l is None or l == "inf" else float(l))

    def to_json(self):
        return [self.retention, None if math.isinf(self.limit) else self.limit]


@dataclass
class LayerSpec:
    elts: List[int]
    occ: Terms  # FT2
    agg: Terms  # FT3


@dataclass
class Config:
    name: str
    num_trials: int
    kmin: int
    kmax: int
    catalog_size: int
    entries_per_elt: int
    elt_terms: List[Terms]  # FT1 per ELT (global ELT index)
    layers: List[LayerSpec]
    regime: str = "real"
    seed: int = SEED
    description: str = ""

    @property
    def num_elts(self) -> int:
        return len(self.elt_terms)

    @property
    def fixed_length(self) -> bool:
        return self.kmin == self.kmax

    @staticmethod
    def load(path_or_name: str) -> "Config":
        path = path_or_name
        if not os.path.exists(path):
            path = os.path.join(os.path.dirname(__file__), "..", "..", "configs", f"{path_or_name}.json")
        with open(path) as f:
            d = json.load(f)
        return Config(
            name=d["name"], num_trials=d["num_trials"], kmin=d["kmin"], kmax=d["kmax"],
            catalog_size=d["catalog_size"], entries_per_elt=d["entries_per_elt"],
            elt_terms=[Terms.from_json(t) for t in d["elt_terms"]],
            layers=[LayerSpec(l["elts"], Terms.from_json(l["occ"]), Terms.from_json(l["agg"])) for l in d["layers"]],
            regime=d.get("regime", "real"), seed=d.get("seed", SEED), description=d.get("description", ""))

    def to_json(self) -> dict:
        return {
            "name": self.name, "description": self.description, "seed": self.seed, "regime": self.regime,
            "num_trials": self.num_trials, "kmin": self.kmin, "kmax": self.kmax,
            "catalog_size": self.catalog_size, "entries_per_elt": self.entries_per_elt,
            "elt_terms": [t.to_json() for t in self.elt_terms],
            "layers": [{"elts": l.elts, "occ": l.occ.to_json(), "agg": l.agg.to_json()} for l in self.layers],
        }


@dataclass
class EltData:
    event_ids: np.ndarray  # uint32
    losses: np.ndarray  # float32
    ft1: Terms


def make_elts(cfg: Config) -> List[EltData]:
    out = []
    for g, t in enumerate(cfg.elt_terms):
        ids = elt_event_ids(cfg.seed, g, cfg.entries_per_elt, cfg.catalog_size)
        losses = elt_losses(cfg.seed, g, cfg.entries_per_elt, cfg.regime)
        out.append(EltData(ids, losses, t))
    return out


@dataclass
class YetData:
    event_ids: np.ndarray  # uint32, trial-major
    offsets: Optional[np.ndarray]  # uint64 [n+1] relative to event_ids[0]; None => fixed length
    num_trials: int
    events_per_trial: int  # when offsets is None


def make_yet(cfg: Config, t0: int = 0, t1: Optional[int] = None) -> YetData:
    """Host YET for trials [t0, t1) of the config (ids of the GLOBAL occurrence range)."""
    t1 = cfg.num_trials if t1 is None else t1
    n = t1 - t0
    if cfg.fixed_length:
        k = cfg.kmin
        ids = yet_ids_chunked(cfg.seed, cfg.catalog_size, t0 * k, n * k)
        return YetData(ids, None, n, k)
    off = trial_offsets(cfg.seed, cfg.num_trials, cfg.kmin, cfg.kmax)
    q0, q1 = int(off[t0]), int(off[t1])
    ids = yet_ids(cfg.seed, cfg.catalog_size, q0, q1 - q0)
    return YetData(ids, (off[t0:t1 + 1] - np.uint64(q0)).astype(np.uint64), n, 0)


def make_yet_trials(cfg: Config, trials: Sequence[int]) -> YetData:
    """Host YET holding only the listed trials (for sampled parity against the oracle)."""
    trials = np.asarray(trials, dtype=np.int64)
    if cfg.fixed_length:
        k = cfg.kmin
        q = (trials[:, None] * k + np.arange(k)[None, :]).reshape(-1)
        r = draws_at(cfg.seed, stream(KIND_YET_IDS), q.astype(np.uint64))
        ids = (uni_np(r, cfg.catalog_size) + np.uint64(1)).astype(np.uint32)
        return YetData(ids, None, len(trials), k)
    off = trial_offsets(cfg.seed, cfg.num_trials, cfg.kmin, cfg.kmax)
    parts, lens = [], []
    for t in trials:
        q0, q1 = int(off[t]), int(off[t + 1])
        parts.append(yet_ids(cfg.seed, cfg.catalog_size, q0, q1 - q0))
        lens.append(q1 - q0)
    o = np.zeros(len(trials) + 1, dtype=np.uint64)
    np.cumsum(np.asarray(lens, dtype=np.uint64), out=o[1:])
    return YetData(np.concatenate(parts) if parts else np.zeros(0, np.uint32), o, len(trials), 0)


# ---------------------------------------------------------------- device generator binding
_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(os.path.dirname(__file__), "libara_synth.so")
        if not os.path.exists(path):
            raise RuntimeError(f"device generator not built: {path} missing (run __graft_entry__.build())")
        lib = ctypes.CDLL(path)
        lib.ara_synth_yet_ids.restype = ctypes.c_int
        lib.ara_synth_yet_ids.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                          ctypes.c_uint32, ctypes.c_void_p]
        lib.ara_synth_last_error.restype = ctypes.c_char_p
        _LIB = lib
    return _LIB


def yet_ids_device(out_ptr: int, seed: int, catalog_size: int, q0: int, count: int, stream_ptr: int) -> None:
    """Fill device buffer out_ptr[0:count] with ids of global occurrences q0.. (async on stream)."""
    st = _lib().ara_synth_yet_ids(out_ptr, seed, q0, count, catalog_size, stream_ptr)
    if st != 0:
        raise RuntimeError(f"ara_synth_yet_ids failed: {_lib().ara_synth_last_error().decode()}")


def return_periods(n: int) -> List[float]:
    """Workload parameter (reading c11): the return periods PML/TVaR are read at --
    {2,5,10,20,25,50,100,200,250,500,1000}, plus {5000,10000} when N >= 1e6; only RP <= N."""
    rps = [2, 5, 10, 20, 25, 50, 100, 200, 250, 500, 1000]
    if n >= 1_000_000:
        rps += [5000, 10000]
    return [float(r) for r in rps if r <= n]
