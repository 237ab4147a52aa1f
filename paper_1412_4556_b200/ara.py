"""Thin Python binding of libara (include/ara.h): argument marshalling only.

Every function here has the name of the C entry point it calls and does no arithmetic of the
method: all compute runs in libara's sm_100a kernels.  There is no fallback -- if libara.so is
missing or the device is not a B200 the call raises.

Inputs: ELTs / layers as host numpy arrays (copied by ara_create); the YET and the YLT as CUDA torch
tensors (ara_run, device path) or pinned host tensors / numpy arrays (ara_run_host, end-to-end path).
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libara.so")

ARA_OK, ARA_E_ARG, ARA_E_RANGE, ARA_E_DUP, ARA_E_VALUE, ARA_E_NOMEM, ARA_E_CUDA, ARA_E_UNSUPPORTED = range(8)
ARA_OPT_BLOCK_THREADS, ARA_OPT_BLOCKS_PER_SM, ARA_OPT_L2_POLICY, ARA_OPT_VARIANT, ARA_OPT_KERNEL = 1, 2, 3, 4, 5
ARA_OPT_PREFETCH = 6
ARA_OPT_FILTER = 7
ARA_OPT_PRECOMBINED = 8
ARA_OPT_STREAM = 9
ARA_OPT_ROUND_MIN = 10
ARA_OPT_TRIAL_ORDER = 11
ARA_OPT_FUSED = 12
KERNEL_AUTO, KERNEL_PRESENCE, KERNEL_DENSE = -1, 0, 1
STUDY_INTERLEAVED, STUDY_INDEPENDENT, STUDY_SORTED, STUDY_HASH, STUDY_INDEX = 0, 1, 2, 3, 4
ARA_MAX_ELTS_PER_LAYER = 128

#: every symbol include/ara.h declares (checked by tests/test_abi.py against the header and the .so)
EXPORTS = ("ara_create", "ara_destroy", "ara_run", "ara_run_ex", "ara_run_host", "ara_run_study", "ara_aal", "ara_ep",
           "ara_sum_layers", "ara_check", "ara_pml_tvar", "ara_pml",
           "ara_tvar", "ara_pml_tvar_device", "ara_table_footprint", "ara_unshard", "ara_set_option", "ara_get_option",
           "ara_layer_info", "ara_layer_stats", "ara_kernel_name", "ara_status_string", "ara_last_error",
           "ara_version", "ara_plan_create", "ara_plan_launch", "ara_plan_destroy", "ara_metrics_plan_create")


class AraError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        self.status = status
        super().__init__(f"{where}: {_status_name(status)}: {detail}")


class _Terms(ctypes.Structure):
    _fields_ = [("retention", ctypes.c_double), ("limit", ctypes.c_double)]


class _Elt(ctypes.Structure):
    _fields_ = [("event_ids", ctypes.c_void_p), ("losses", ctypes.c_void_p), ("num_entries", ctypes.c_uint64),
                ("ft1", _Terms)]


class _Layer(ctypes.Structure):
    _fields_ = [("elt_index", ctypes.c_void_p), ("num_elts", ctypes.c_uint32), ("occurrence", _Terms),
                ("aggregate", _Terms)]


class _Yet(ctypes.Structure):
    _fields_ = [("event_ids", ctypes.c_void_p), ("trial_offsets", ctypes.c_void_p), ("num_trials", ctypes.c_uint64),
                ("num_events", ctypes.c_uint64), ("events_per_trial", ctypes.c_uint32)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libara.so (in-tree).  Raises if it has not been built -- there is no fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        st, vp, u32, u64, dp = ctypes.c_int, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p
        sig = {
            "ara_create": (st, [u32, ctypes.POINTER(_Elt), u32, ctypes.POINTER(_Layer), u32, ctypes.c_int, vp,
                                ctypes.POINTER(vp)]),
            "ara_destroy": (None, [vp]),
            "ara_run": (st, [vp, ctypes.POINTER(_Yet), dp, vp]),
            "ara_run_host": (st, [vp, ctypes.POINTER(_Yet), dp, vp]),
            "ara_run_ex": (st, [vp, ctypes.POINTER(_Yet), dp, dp, vp]),
            "ara_aal": (st, [dp, u64, dp, vp]),
            "ara_ep": (st, [dp, u64, dp, u32, dp, vp]),
            "ara_sum_layers": (st, [dp, u32, u64, dp, u32, dp, vp]),
            "ara_run_study": (st, [vp, ctypes.c_int, ctypes.POINTER(_Yet), dp, vp]),
            "ara_check": (st, [vp, vp]),
            "ara_pml_tvar": (st, [dp, u64, dp, u32, dp, dp, vp]),
            "ara_pml": (st, [dp, u64, dp, u32, dp, vp]),
            "ara_pml_tvar_device": (st, [dp, u64, dp, u32, dp, dp, vp]),
            "ara_tvar": (st, [dp, u64, dp, u32, dp, vp]),
            "ara_table_footprint": (st, [u32, u32, ctypes.POINTER(u64), ctypes.POINTER(u32)]),
            "ara_unshard": (st, [dp, u32, u64, u32, dp, dp, vp]),
            "ara_set_option": (st, [vp, ctypes.c_int, ctypes.c_int64]),
            "ara_get_option": (st, [vp, ctypes.c_int, ctypes.POINTER(ctypes.c_int64)]),
            "ara_layer_info": (st, [vp, u32, ctypes.POINTER(u64), ctypes.POINTER(u32), ctypes.POINTER(u32),
                                    ctypes.POINTER(ctypes.c_char_p)]),
            "ara_layer_stats": (st, [vp, u32, ctypes.POINTER(u64), ctypes.POINTER(ctypes.c_double),
                                     ctypes.POINTER(ctypes.c_int)]),
            "ara_kernel_name": (ctypes.c_char_p, [vp]),
            "ara_plan_create": (st, [vp, ctypes.POINTER(_Yet), dp, dp, u32, dp, dp, vp, ctypes.POINTER(vp)]),
            "ara_plan_launch": (st, [vp, vp]),
            "ara_plan_destroy": (None, [vp]),
            "ara_metrics_plan_create": (st, [dp, u64, u32, dp, u32, dp, dp, u64, vp, ctypes.POINTER(vp)]),
            "ara_status_string": (ctypes.c_char_p, [ctypes.c_int]),
            "ara_last_error": (ctypes.c_char_p, []),
            "ara_version": (u32, []),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


TESTING_LIB_PATH = os.path.join(_HERE, "libara_testing.so")
TESTING_EXPORTS = ("ara_table_row", "ara_testing_last_error")
_tlib = None


def testing_lib() -> ctypes.CDLL:
    """Load the test-only libara_testing.so (include/ara_testing.h); libara.so is loaded first."""
    global _tlib
    if _tlib is None:
        lib()
        if not os.path.exists(TESTING_LIB_PATH):
            raise RuntimeError(f"{TESTING_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        T = ctypes.CDLL(TESTING_LIB_PATH)
        T.ara_table_row.restype = ctypes.c_int
        T.ara_table_row.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p]
        T.ara_testing_last_error.restype = ctypes.c_char_p
        T.ara_testing_last_error.argtypes = []
        _tlib = T
    return _tlib


def _status_name(s: int) -> str:
    try:
        return lib().ara_status_string(s).decode()
    except Exception:  # noqa: BLE001
        return str(s)


def _check(status: int, where: str) -> None:
    if status != ARA_OK:
        raise AraError(status, where, lib().ara_last_error().decode())


def _stream_ptr(stream) -> int:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _dptr(t) -> int:
    """Data pointer of a torch tensor (device or host) or numpy array."""
    if t is None:
        return 0
    if isinstance(t, np.ndarray):
        return t.ctypes.data if t.size else 0
    return t.data_ptr()


# ---------------------------------------------------------------------------------------- inputs
@dataclass
class Elt:
    event_ids: np.ndarray  # uint32
    losses: np.ndarray  # float32
    retention: float = 0.0
    limit: float = math.inf


@dataclass
class Layer:
    elts: Sequence[int]
    occ_retention: float = 0.0
    occ_limit: float = math.inf
    agg_retention: float = 0.0
    agg_limit: float = math.inf


def ara_version() -> Tuple[int, int]:
    v = lib().ara_version()
    return v >> 16, v & 0xFFFF


def ara_table_footprint(catalog_size: int, num_elts: int) -> Tuple[int, int]:
    b, s = ctypes.c_uint64(), ctypes.c_uint32()
    _check(lib().ara_table_footprint(catalog_size, num_elts, ctypes.byref(b), ctypes.byref(s)), "ara_table_footprint")
    return b.value, s.value


def _yet_struct(event_ids, offsets, num_trials: int, events_per_trial: int):
    n_ev = int(event_ids.numel() if hasattr(event_ids, "numel") else event_ids.size)
    return _Yet(_dptr(event_ids), _dptr(offsets), num_trials, n_ev, events_per_trial)


class Context:
    """Owns an ara_ctx: one per device (rank).  Methods map 1:1 onto the C entry points."""

    def __init__(self, catalog_size: int, elts: Sequence[Elt], layers: Sequence[Layer], device: int = 0,
                 stream=None):
        keep = []
        ce = (_Elt * max(1, len(elts)))()
        for j, e in enumerate(elts):
            ids = np.ascontiguousarray(e.event_ids, dtype=np.uint32)
            losses = np.ascontiguousarray(e.losses, dtype=np.float32)
            if ids.shape != losses.shape:
                raise ValueError(f"ELT {j}: ids and losses differ in length")
            keep += [ids, losses]
            ce[j] = _Elt(_dptr(ids), _dptr(losses), ids.size, _Terms(e.retention, e.limit))
        cl = (_Layer * max(1, len(layers)))()
        for l, L in enumerate(layers):
            idx = np.ascontiguousarray(L.elts, dtype=np.uint32)
            keep.append(idx)
            cl[l] = _Layer(_dptr(idx), idx.size, _Terms(L.occ_retention, L.occ_limit),
                           _Terms(L.agg_retention, L.agg_limit))
        h = ctypes.c_void_p()
        s = _stream_ptr(stream) if stream is not None or _torch_cuda() else 0
        _check(lib().ara_create(catalog_size, ce, len(elts), cl, len(layers), device, s, ctypes.byref(h)), "ara_create")
        self._h = h
        self.device = device
        self.num_layers = len(layers)
        self.catalog_size = catalog_size

    # -- lifetime
    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().ara_destroy(self._h)
            self._h = None

    ara_destroy = close

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- the hot path
    def ara_run(self, event_ids, ylt, offsets=None, events_per_trial: int = 0, num_trials: Optional[int] = None,
                stream=None) -> None:
        """Device YET (CUDA uint32 tensor) -> device YLT (CUDA float64 tensor [layers, trials]).  Async."""
        n = num_trials if num_trials is not None else (offsets.numel() - 1 if offsets is not None else
                                                       event_ids.numel() // max(1, events_per_trial))
        y = _yet_struct(event_ids, offsets, n, events_per_trial)
        _check(lib().ara_run(self._h, ctypes.byref(y), _dptr(ylt), _stream_ptr(stream)), "ara_run")

    def ara_plan_create(self, event_ids, ylt, rps, pml_dev=None, tvar_dev=None, offsets=None,
                        events_per_trial: int = 0, num_trials: Optional[int] = None, stream=None) -> "Plan":
        """Capture one analysis step (ara_run + PML/TVaR of every layer into device [layers, m] buffers)
        as a CUDA graph; returns a Plan whose launch() replays it.  The tensors must outlive the plan."""
        n = num_trials if num_trials is not None else (offsets.numel() - 1 if offsets is not None else
                                                       event_ids.numel() // max(1, events_per_trial))
        y = _yet_struct(event_ids, offsets, n, events_per_trial)
        r = np.ascontiguousarray(rps, dtype=np.float64)
        h = ctypes.c_void_p()
        _check(lib().ara_plan_create(self._h, ctypes.byref(y), _dptr(ylt), _dptr(r), r.size, _dptr(pml_dev),
                                     _dptr(tvar_dev), _stream_ptr(stream), ctypes.byref(h)), "ara_plan_create")
        return Plan(h, (event_ids, ylt, offsets, pml_dev, tvar_dev, r, self))

    def ara_run_ex(self, event_ids, ylt, olt=None, offsets=None, events_per_trial: int = 0,
                   num_trials: Optional[int] = None, stream=None) -> None:
        """ara_run plus the occurrence-basis table (largest occurrence-net loss per trial)."""
        n = num_trials if num_trials is not None else (offsets.numel() - 1 if offsets is not None else
                                                       event_ids.numel() // max(1, events_per_trial))
        y = _yet_struct(event_ids, offsets, n, events_per_trial)
        _check(lib().ara_run_ex(self._h, ctypes.byref(y), _dptr(ylt), _dptr(olt), _stream_ptr(stream)), "ara_run_ex")

    def ara_run_host(self, event_ids, ylt_host, offsets=None, events_per_trial: int = 0,
                     num_trials: Optional[int] = None, stream=None) -> None:
        """Host YET (pinned for overlap) -> host YLT.  Synchronous, includes the validity check."""
        n = num_trials if num_trials is not None else (len(offsets) - 1 if offsets is not None else
                                                       _numel(event_ids) // max(1, events_per_trial))
        y = _yet_struct(event_ids, offsets, n, events_per_trial)
        _check(lib().ara_run_host(self._h, ctypes.byref(y), _dptr(ylt_host), _stream_ptr(stream)), "ara_run_host")

    def ara_run_study(self, layout: int, event_ids, ylt, offsets=None, events_per_trial: int = 0,
                      num_trials: Optional[int] = None, stream=None) -> None:
        """Section IV.B data-structure study kernel (device YET -> device YLT)."""
        n = num_trials if num_trials is not None else (offsets.numel() - 1 if offsets is not None else
                                                       event_ids.numel() // max(1, events_per_trial))
        y = _yet_struct(event_ids, offsets, n, events_per_trial)
        _check(lib().ara_run_study(self._h, layout, ctypes.byref(y), _dptr(ylt), _stream_ptr(stream)), "ara_run_study")

    def ara_check(self, stream=None) -> None:
        _check(lib().ara_check(self._h, _stream_ptr(stream)), "ara_check")

    # -- knobs / introspection
    def ara_set_option(self, opt: int, value: int) -> None:
        _check(lib().ara_set_option(self._h, opt, value), "ara_set_option")

    def ara_get_option(self, opt: int) -> int:
        v = ctypes.c_int64()
        _check(lib().ara_get_option(self._h, opt, ctypes.byref(v)), "ara_get_option")
        return v.value

    def ara_layer_info(self, layer: int = 0) -> dict:
        b, s, nv, name = ctypes.c_uint64(), ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_char_p()
        _check(lib().ara_layer_info(self._h, layer, ctypes.byref(b), ctypes.byref(s), ctypes.byref(nv),
                                    ctypes.byref(name)), "ara_layer_info")
        return {"table_bytes": b.value, "row_stride": s.value, "num_variants": nv.value, "variant": name.value.decode()}

    def ara_layer_stats(self, layer: int = 0) -> dict:
        pr, hr, k = ctypes.c_uint64(), ctypes.c_double(), ctypes.c_int()
        _check(lib().ara_layer_stats(self._h, layer, ctypes.byref(pr), ctypes.byref(hr), ctypes.byref(k)),
               "ara_layer_stats")
        return {"present_rows": pr.value, "est_hit_rate": hr.value, "kernel": k.value}

    def ara_kernel_name(self) -> str:
        """Kernel the last run launched (for reports)."""
        return lib().ara_kernel_name(self._h).decode()

    def ara_table_row(self, layer: int, event: int) -> np.ndarray:
        """Test hook (libara_testing.so, include/ara_testing.h): row `event` of layer `layer`'s table."""
        stride = self.ara_layer_info(layer)["row_stride"]
        out = np.zeros(stride // 4, dtype=np.float32)
        T = testing_lib()
        st = T.ara_table_row(self._h, layer, event, _dptr(out))
        if st != ARA_OK:
            raise AraError(st, "ara_table_row", T.ara_testing_last_error().decode())
        return out


class Plan:
    """A captured analysis step (ara_plan_create); launch() = one CUDA graph launch."""

    def __init__(self, handle, keep):
        self._h = handle
        self._keep = keep  # the buffers the graph reads and writes stay alive with the plan

    def launch(self, stream=None) -> None:
        _check(lib().ara_plan_launch(self._h, _stream_ptr(stream)), "ara_plan_launch")

    def close(self) -> None:
        if self._h:
            lib().ara_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def _numel(a) -> int:
    return int(a.numel()) if hasattr(a, "numel") else int(a.size)


def _torch_cuda() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        return False


def ara_pml_tvar(ylt, rps: Sequence[float], stream=None, n: Optional[int] = None) -> Tuple[np.ndarray, np.ndarray]:
    """PML and TVaR of a device YLT (1-D CUDA float64 tensor or its first n values)."""
    r = np.ascontiguousarray(rps, dtype=np.float64)
    pml = np.zeros(max(1, r.size))
    tv = np.zeros(max(1, r.size))
    n = _numel(ylt) if n is None else n
    _check(lib().ara_pml_tvar(_dptr(ylt), n, _dptr(r), r.size, _dptr(pml), _dptr(tv), _stream_ptr(stream)),
           "ara_pml_tvar")
    return pml[:r.size], tv[:r.size]


def ara_pml_tvar_device(ylt, rps: Sequence[float], pml_dev, tvar_dev, stream=None, n: Optional[int] = None) -> None:
    """Asynchronous PML/TVaR into CUDA float64 tensors pml_dev / tvar_dev (len(rps) each, either None)."""
    r = np.ascontiguousarray(rps, dtype=np.float64)
    n = _numel(ylt) if n is None else n
    _check(lib().ara_pml_tvar_device(_dptr(ylt), n, _dptr(r), r.size, _dptr(pml_dev), _dptr(tvar_dev),
                                     _stream_ptr(stream)), "ara_pml_tvar_device")


def ara_metrics_plan_create(ylt, rps: Sequence[float], pml_dev=None, tvar_dev=None, out_stride: Optional[int] = None,
                            stream=None) -> "Plan":
    """Capture PML/TVaR of a device YLT [layers, n] (or [n]) as a CUDA graph (ara_metrics_plan_create); layer
    l's results land at pml_dev / tvar_dev + l * out_stride (default m).  The tensors must outlive the plan."""
    r = np.ascontiguousarray(rps, dtype=np.float64)
    layers, n = (1, ylt.numel()) if ylt.dim() == 1 else (ylt.shape[0], ylt.shape[1])
    h = ctypes.c_void_p()
    _check(lib().ara_metrics_plan_create(_dptr(ylt), n, layers, _dptr(r), r.size, _dptr(pml_dev), _dptr(tvar_dev),
                                         out_stride if out_stride is not None else r.size, _stream_ptr(stream),
                                         ctypes.byref(h)), "ara_metrics_plan_create")
    return Plan(h, (ylt, pml_dev, tvar_dev, r))


def ara_pml(ylt, rps: Sequence[float], stream=None) -> np.ndarray:
    r = np.ascontiguousarray(rps, dtype=np.float64)
    out = np.zeros(max(1, r.size))
    _check(lib().ara_pml(_dptr(ylt), _numel(ylt), _dptr(r), r.size, _dptr(out), _stream_ptr(stream)), "ara_pml")
    return out[:r.size]


def ara_tvar(ylt, rps: Sequence[float], stream=None) -> np.ndarray:
    r = np.ascontiguousarray(rps, dtype=np.float64)
    out = np.zeros(max(1, r.size))
    _check(lib().ara_tvar(_dptr(ylt), _numel(ylt), _dptr(r), r.size, _dptr(out), _stream_ptr(stream)), "ara_tvar")
    return out[:r.size]


def ara_aal(ylt, stream=None, n: Optional[int] = None) -> float:
    out = ctypes.c_double()
    _check(lib().ara_aal(_dptr(ylt), _numel(ylt) if n is None else n, ctypes.addressof(out), _stream_ptr(stream)),
           "ara_aal")
    return out.value


def ara_ep(ylt, thresholds: Sequence[float], stream=None) -> np.ndarray:
    x = np.ascontiguousarray(thresholds, dtype=np.float64)
    out = np.zeros(max(1, x.size))
    _check(lib().ara_ep(_dptr(ylt), _numel(ylt), _dptr(x), x.size, _dptr(out), _stream_ptr(stream)), "ara_ep")
    return out[:x.size]


def ara_sum_layers(ylt, group: Sequence[int], num_groups: int, out, stream=None) -> None:
    """ylt: CUDA [layers, n]; out: CUDA [num_groups, n]."""
    g = np.ascontiguousarray(group, dtype=np.uint32)
    _check(lib().ara_sum_layers(_dptr(ylt), g.size, ylt.shape[1], _dptr(g), num_groups, _dptr(out),
                                _stream_ptr(stream)), "ara_sum_layers")


def ara_unshard(gathered, num_shards: int, shard_cap: int, num_layers: int, starts: Sequence[int], ylt,
                stream=None) -> None:
    s = np.ascontiguousarray(starts, dtype=np.uint64)
    _check(lib().ara_unshard(_dptr(gathered), num_shards, shard_cap, num_layers, _dptr(s), _dptr(ylt),
                             _stream_ptr(stream)), "ara_unshard")


# ---------------------------------------------------------------------------------------- config glue
def context_for_config(cfg, elt_data, device: int = 0, stream=None) -> Context:
    """Build a Context from a synth.Config and its generated ELTs."""
    elts = [Elt(e.event_ids, e.losses, e.ft1.retention, e.ft1.limit) for e in elt_data]
    layers = [Layer(l.elts, l.occ.retention, l.occ.limit, l.agg.retention, l.agg.limit) for l in cfg.layers]
    return Context(cfg.catalog_size, elts, layers, device=device, stream=stream)
