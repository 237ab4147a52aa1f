"""CPU-only checks of the C-ABI boundary: the library loads, exports exactly what include/ara.h
declares, and its host-side validation / accounting behave as documented.  No compute calls."""
import math
import os
import re
import subprocess

import numpy as np
import pytest

from ara_testutil import ROOT, golden
from paper_1412_4556_b200 import ara

HEADER = os.path.join(ROOT, "include", "ara.h")


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"ARA_API\s+[\w\s\*]+?\b(ara_\w+)\s*\(", txt)))


def test_header_declares_binding_exports():
    assert _declared() == sorted(ara.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = ara.lib()
    for name in _declared():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", ara.LIB_PATH], capture_output=True, text=True).stdout
    exported = sorted(l.split()[-1] for l in out.splitlines() if " T " in l)
    assert exported == _declared()


def test_testing_library_exports_its_header():
    """Test hooks live in libara_testing.so (include/ara_testing.h), not in the product ABI."""
    txt = open(os.path.join(ROOT, "include", "ara_testing.h")).read()
    declared = sorted(set(re.findall(r"ARA_API\s+[\w\s\*]+?\b(ara_\w+)\s*\(", txt)))
    assert declared == sorted(ara.TESTING_EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", ara.TESTING_LIB_PATH], capture_output=True, text=True).stdout
    assert sorted(l.split()[-1] for l in out.splitlines() if " T " in l) == declared
    assert "ara_table_row" not in _declared()
    T = ara.testing_lib()
    assert T.ara_table_row(None, 0, 0, None) == ara.ARA_E_ARG


def test_synth_library_exports():
    out = subprocess.run(["nm", "-D", "--defined-only",
                          os.path.join(ROOT, "paper_1412_4556_b200", "synth", "libara_synth.so")],
                         capture_output=True, text=True).stdout
    assert {"ara_synth_yet_ids", "ara_synth_last_error"} <= {l.split()[-1] for l in out.splitlines() if " T " in l}


def test_version_and_status_strings():
    assert ara.ara_version() == (0, 2)
    names = [ara.lib().ara_status_string(i).decode() for i in range(8)]
    assert names == ["ARA_OK", "ARA_E_ARG", "ARA_E_RANGE", "ARA_E_DUP", "ARA_E_VALUE", "ARA_E_NOMEM", "ARA_E_CUDA",
                     "ARA_E_UNSUPPORTED"]


def test_table_footprint_pins_paper_memory_accounting():
    """15 ELTs x 1M-event catalogue -> 15M event-loss pairs, 14,850,000 of them zero."""
    g = golden("memory_accounting.json")
    for c in g["cases"]:
        C, J, n = c["catalog"], c["num_elts"], c["entries"]
        assert J * C == c["pairs"]
        assert J * (C - n) == c["zero_entries"]
        b, stride = ara.ara_table_footprint(C, J)
        assert b == (C + 1) * stride
        if "table_bytes" in c:
            assert (b, stride) == (c["table_bytes"], c["row_stride"])


def test_row_stride_never_straddles_sectors():
    for J in range(1, 129):
        _, s = ara.ara_table_footprint(1000, J)
        assert s >= 4 * J
        if 4 * J <= 32:
            assert s & (s - 1) == 0 and 32 % s == 0
        else:
            assert s % 32 == 0 and s - 4 * J < 32


def _ctx(elts, layers, C=10):
    return ara.Context(C, elts, layers, device=0, stream=0)


GOOD = [ara.Elt(np.array([1, 2], np.uint32), np.array([5.0, 6.0], np.float32), 1.0, 10.0)]


@pytest.mark.parametrize("elts,layers,status", [
    ([ara.Elt(np.array([0], np.uint32), np.array([1.0], np.float32))], [ara.Layer([0])], ara.ARA_E_RANGE),
    ([ara.Elt(np.array([11], np.uint32), np.array([1.0], np.float32))], [ara.Layer([0])], ara.ARA_E_RANGE),
    ([ara.Elt(np.array([3, 3], np.uint32), np.array([1.0, 2.0], np.float32))], [ara.Layer([0])], ara.ARA_E_DUP),
    ([ara.Elt(np.array([3], np.uint32), np.array([0.0], np.float32))], [ara.Layer([0])], ara.ARA_E_VALUE),
    ([ara.Elt(np.array([3], np.uint32), np.array([np.inf], np.float32))], [ara.Layer([0])], ara.ARA_E_VALUE),
    ([ara.Elt(np.array([3], np.uint32), np.array([np.nan], np.float32))], [ara.Layer([0])], ara.ARA_E_VALUE),
    ([ara.Elt(np.array([3], np.uint32), np.array([1.0], np.float32), -1.0)], [ara.Layer([0])], ara.ARA_E_VALUE),
    ([ara.Elt(np.array([3], np.uint32), np.array([1.0], np.float32), 0.0, 0.0)], [ara.Layer([0])], ara.ARA_E_VALUE),
    (GOOD, [ara.Layer([0], occ_limit=math.nan)], ara.ARA_E_VALUE),
    (GOOD, [ara.Layer([0], agg_retention=math.inf)], ara.ARA_E_VALUE),
    (GOOD, [ara.Layer([1])], ara.ARA_E_ARG),
    (GOOD, [ara.Layer([0, 0])], ara.ARA_E_ARG),
    (GOOD, [ara.Layer([])], ara.ARA_E_ARG),
    (GOOD, [], ara.ARA_E_ARG),
    ([], [ara.Layer([0])], ara.ARA_E_ARG),
])
def test_create_validation_errors(elts, layers, status):
    """Host validation runs before any device call (SPEC.md:29-58 invariants)."""
    with pytest.raises(ara.AraError) as ei:
        _ctx(elts, layers)
    assert ei.value.status == status


def test_too_many_elts_per_layer_unsupported():
    elts = [ara.Elt(np.array([1], np.uint32), np.array([1.0], np.float32)) for _ in range(129)]
    with pytest.raises(ara.AraError) as ei:
        _ctx(elts, [ara.Layer(list(range(129)))])
    assert ei.value.status == ara.ARA_E_UNSUPPORTED


@pytest.mark.parametrize("rps,status", [([1.0], ara.ARA_E_RANGE), ([0.5], ara.ARA_E_RANGE), ([11.0], ara.ARA_E_RANGE),
                                        ([math.nan], ara.ARA_E_RANGE), ([], ara.ARA_E_ARG)])
def test_metric_argument_validation(rps, status):
    """Return periods are checked on the host before the device is touched (readings c11, c12)."""
    with pytest.raises(ara.AraError) as ei:
        ara.ara_pml_tvar(np.zeros(10), rps, stream=0, n=10)
    assert ei.value.status == status


def test_no_cpu_fallback_in_product_package():
    """The product package never imports the oracle and has no host compute path."""
    pkg = os.path.join(ROOT, "paper_1412_4556_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
