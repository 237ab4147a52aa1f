"""CPU oracle for Aggregate Risk Analysis -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference`` legs may
import this package.  The product path (paper_1412_4556_b200) never imports it, and it never
imports the product path.  See ara_oracle.h for what it computes and which PAPER.md passages each
step follows; DESIGN.md lists the readings (c1..c22) it implements.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libara_oracle.so")
_SRC = os.path.join(_HERE, "ara_oracle.c")

LOOKUP_BINARY = 0
LOOKUP_LINEAR = 1


def build(force: bool = False) -> str:
    """Compile the oracle (plain C, fp64, no FMA contraction)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "ara_oracle.h"))):
        cmd = ["gcc", "-std=c99", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-pthread",
               "-o", _SO, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _SO


class _Elt(ctypes.Structure):
    _fields_ = [("event_ids", ctypes.c_void_p), ("losses", ctypes.c_void_p), ("n", ctypes.c_uint64),
                ("ft1_retention", ctypes.c_double), ("ft1_limit", ctypes.c_double)]


class _Layer(ctypes.Structure):
    _fields_ = [("elt_index", ctypes.c_void_p), ("num_elts", ctypes.c_uint32),
                ("ft2_retention", ctypes.c_double), ("ft2_limit", ctypes.c_double),
                ("ft3_retention", ctypes.c_double), ("ft3_limit", ctypes.c_double)]


_lib = None


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        lib.oracle_clamp.restype = ctypes.c_double
        lib.oracle_clamp.argtypes = [ctypes.c_double] * 3
        lib.oracle_ylt.restype = ctypes.c_int
        lib.oracle_ylt.argtypes = [ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                   ctypes.c_uint32, ctypes.POINTER(_Elt), ctypes.c_uint32,
                                   ctypes.POINTER(_Layer), ctypes.c_uint32, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_void_p]
        lib.oracle_ylt_olt.restype = ctypes.c_int
        lib.oracle_ylt_olt.argtypes = lib.oracle_ylt.argtypes + [ctypes.c_void_p]
        lib.oracle_aal.restype = ctypes.c_double
        lib.oracle_aal.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
        lib.oracle_ep.restype = None
        lib.oracle_ep.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p]
        lib.oracle_trial_detail.restype = ctypes.c_int
        lib.oracle_trial_detail.argtypes = [ctypes.c_uint32, ctypes.c_void_p, ctypes.c_uint64,
                                            ctypes.POINTER(_Elt), ctypes.c_uint32, ctypes.POINTER(_Layer),
                                            ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                            ctypes.c_void_p]
        lib.oracle_rank.restype = ctypes.c_uint64
        lib.oracle_rank.argtypes = [ctypes.c_uint64, ctypes.c_double]
        for f in (lib.oracle_pml, lib.oracle_tvar):
            f.restype = ctypes.c_int
            f.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p]
        lib.oracle_default_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


class OracleError(RuntimeError):
    pass


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data if a.size else 0


def clamp(x: float, retention: float, limit: float) -> float:
    return _L().oracle_clamp(x, retention, limit)


def default_threads() -> int:
    return _L().oracle_default_threads()


def _marshal(elts, layers):
    """elts: sequence of (ids uint32, losses float32, (R1, L1)); layers: sequence of
    (elt index list, (R2, L2), (R3, L3)).  Returns ctypes arrays plus keep-alive list."""
    keep = []
    ce = (_Elt * max(1, len(elts)))()
    for j, (ids, losses, ft1) in enumerate(elts):
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        losses = np.ascontiguousarray(losses, dtype=np.float32)
        if ids.shape != losses.shape:
            raise ValueError("ELT ids/losses length mismatch")
        keep += [ids, losses]
        ce[j] = _Elt(_ptr(ids), _ptr(losses), ids.size, float(ft1[0]), float(ft1[1]))
    cl = (_Layer * max(1, len(layers)))()
    for l, (idx, ft2, ft3) in enumerate(layers):
        idx = np.ascontiguousarray(idx, dtype=np.uint32)
        keep.append(idx)
        cl[l] = _Layer(_ptr(idx), idx.size, float(ft2[0]), float(ft2[1]), float(ft3[0]), float(ft3[1]))
    return ce, cl, keep


def ylt(catalog_size: int, yet_ids: np.ndarray, offsets: Optional[np.ndarray], num_trials: int,
        events_per_trial: int, elts, layers, lookup: int = LOOKUP_BINARY, threads: int = 0) -> np.ndarray:
    """Algorithm 1 over all layers; returns YLT [num_layers][num_trials] float64."""
    yet_ids = np.ascontiguousarray(yet_ids, dtype=np.uint32)
    off = None if offsets is None else np.ascontiguousarray(offsets, dtype=np.uint64)
    ce, cl, keep = _marshal(elts, layers)
    out = np.zeros((len(layers), num_trials), dtype=np.float64)
    rc = _L().oracle_ylt(catalog_size, _ptr(yet_ids), 0 if off is None else _ptr(off), num_trials,
                         events_per_trial, ce, len(elts), cl, len(layers), lookup, threads, _ptr(out))
    if rc:
        raise OracleError(f"oracle_ylt failed with code {rc}")
    return out


def ylt_olt(catalog_size: int, yet_ids: np.ndarray, offsets: Optional[np.ndarray], num_trials: int,
            events_per_trial: int, elts, layers, lookup: int = LOOKUP_BINARY, threads: int = 0):
    """(YLT, OLT): OLT[l][t] = largest occurrence-net loss of trial t under layer l."""
    yet_ids = np.ascontiguousarray(yet_ids, dtype=np.uint32)
    off = None if offsets is None else np.ascontiguousarray(offsets, dtype=np.uint64)
    ce, cl, keep = _marshal(elts, layers)
    y = np.zeros((len(layers), num_trials), dtype=np.float64)
    o = np.zeros((len(layers), num_trials), dtype=np.float64)
    rc = _L().oracle_ylt_olt(catalog_size, _ptr(yet_ids), 0 if off is None else _ptr(off), num_trials,
                             events_per_trial, ce, len(elts), cl, len(layers), lookup, threads, _ptr(y), _ptr(o))
    if rc:
        raise OracleError(f"oracle_ylt_olt failed with code {rc}")
    return y, o


def aal(y: np.ndarray) -> float:
    y = np.ascontiguousarray(y, dtype=np.float64)
    return _L().oracle_aal(_ptr(y), y.size)


def ep(y: np.ndarray, thresholds: Sequence[float]) -> np.ndarray:
    y = np.ascontiguousarray(y, dtype=np.float64)
    x = np.ascontiguousarray(thresholds, dtype=np.float64)
    out = np.zeros(max(1, x.size))
    _L().oracle_ep(_ptr(y), y.size, _ptr(x), x.size, _ptr(out))
    return out[:x.size]


def layer_totals(ylt: np.ndarray, group: Sequence[int], num_groups: int) -> np.ndarray:
    """Program / portfolio totals: out[g][t] = sum of ylt[l][t] over layers l of group g, in layer
    order.  Plain loop."""
    out = np.zeros((num_groups, ylt.shape[1]))
    for l, g in enumerate(group):
        out[g] = out[g] + ylt[l]
    return out


def trial_detail(catalog_size: int, ids: Sequence[int], elts, layer, lookup: int = LOOKUP_BINARY):
    """(o, S, a, ylt) for one trial under one layer."""
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    ce, cl, keep = _marshal(elts, [layer])
    n = ids.size
    o, S, a = (np.zeros(max(n, 1)) for _ in range(3))
    y = ctypes.c_double(0.0)
    rc = _L().oracle_trial_detail(catalog_size, _ptr(ids), n, ce, len(elts), cl, lookup, _ptr(o), _ptr(S),
                                  _ptr(a), ctypes.addressof(y))
    if rc:
        raise OracleError(f"oracle_trial_detail failed with code {rc}")
    return o[:n], S[:n], a[:n], y.value


def rank(n: int, rp: float) -> int:
    return int(_L().oracle_rank(n, rp))


def _metric(fn, y: np.ndarray, rps: Sequence[float]) -> np.ndarray:
    y = np.ascontiguousarray(y, dtype=np.float64)
    r = np.ascontiguousarray(rps, dtype=np.float64)
    out = np.zeros(max(1, r.size))
    rc = fn(_ptr(y), y.size, _ptr(r), r.size, _ptr(out))
    if rc:
        raise OracleError(f"metric failed with code {rc}")
    return out[:r.size]


def pml(y: np.ndarray, rps: Sequence[float]) -> np.ndarray:
    return _metric(_L().oracle_pml, y, rps)


def tvar(y: np.ndarray, rps: Sequence[float]) -> np.ndarray:
    return _metric(_L().oracle_tvar, y, rps)


# ---- convenience over a synth.Config (inputs come from the shared generator module only) -------
def config_elts(cfg, elt_data):
    return [(e.event_ids, e.losses, (e.ft1.retention, e.ft1.limit)) for e in elt_data]


def config_layers(cfg):
    return [(l.elts, (l.occ.retention, l.occ.limit), (l.agg.retention, l.agg.limit)) for l in cfg.layers]


def ylt_for(cfg, elt_data, yet, threads: int = 0, lookup: int = LOOKUP_BINARY) -> np.ndarray:
    return ylt(cfg.catalog_size, yet.event_ids, yet.offsets, yet.num_trials, yet.events_per_trial,
               config_elts(cfg, elt_data), config_layers(cfg), lookup=lookup, threads=threads)


INF = math.inf
