"""CPU: the C-ABI library loads, exports every symbol include/*.h declares,
its host-side helpers work, and every compute entry point refuses to run
without a CUDA device (no CPU fallback)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import kats
import paper_2301_08695_b200 as bx
from conftest import ROOT, cuda_available


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "baechi_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bx_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = bx.lib()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(bx.EXPORTED)


def test_version_string():
    assert b"sm_100a" in bx.lib().bx_version()


@pytest.mark.parametrize("cmb,nbytes,want", kats.COMM_KATS)
def test_host_comm_time_matches_reference_kats(cmb, nbytes, want):
    assert bx.comm_time(bx.CommModel(cmb[0], cmb[1]), nbytes) == want


def test_comm_time_negative_bytes():
    with pytest.raises(bx.ValidationError):
        bx.comm_time(bx.CommModel(1.0, 1.0), -1)


def test_comm_time_matches_oracle_over_many_sizes():
    from oracle import Restate
    rng = np.random.default_rng(0)
    for ic, pb in [(12.5, 0.002), (5.0, 0.001), (0.3, 0.37), (100.0, 0.01)]:
        for b in rng.integers(0, 1 << 26, 200).tolist() + [0, 1, 250, 1 << 30]:
            assert bx.comm_time(bx.CommModel(ic, pb), b) == Restate.comm_time(ic, pb, b)


def test_adjacency_matches_groupedgraph_lists():
    g = kats.diamond()
    m = bx.MetaGraph.from_dict(g)
    assert m.in_off.tolist() == [0, 0, 1, 2, 4]
    assert m.in_edge[:4].tolist() == [0, 1, 2, 3]
    assert m.out_off.tolist() == [0, 2, 3, 4, 4]


def test_adjacency_rejects_unsorted_edges():
    with pytest.raises(bx.ValidationError):
        bx.MetaGraph([1, 1], [0, 0], [0, 0], [0, 0], [1, 0], [0, 1], [0, 0])


@pytest.mark.skipif(cuda_available(), reason="this host has a GPU")
def test_no_cpu_fallback_without_gpu():
    g = bx.MetaGraph.from_dict(kats.diamond())
    with pytest.raises(bx.DeviceError) as ei:
        bx.place_metf(g, [100, 100], bx.CommModel())
    assert "no CPU fallback" in str(ei.value)
    with pytest.raises(bx.DeviceError):
        bx.round_and_extract(2, [0], [1], [0.0])
    with pytest.raises(bx.DeviceError):
        bx.Plan([g], [bx.Job(0, "m-etf", np.array([100, 100]), bx.CommModel())])
    with pytest.raises(bx.DeviceError):
        bx.critical_path_us(g)
    with pytest.raises(bx.DeviceError):
        bx.schedulable_time(bx.PlacerState(g.V, 2, bx.PARALLEL), 3, 0, g, bx.CommModel(0.0, 0.0, bx.PARALLEL))


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2301_08695_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "librestate" not in txt and "libdagsched_ref" not in txt, f
