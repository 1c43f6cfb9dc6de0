"""CPU-side checks of the C ABI library and the host logic (no GPU needed).

* libdpp.so loads and exports every function declared in include/dpp.h;
* the native mesh builder (host C++ inside libdpp) reproduces the reference
  numbering bit-for-bit (golden fixtures) -- it needs no device;
* the option grammar mirrors the reference parser (blocksolve.py:119-210);
* compute entry points fail loudly (no CPU fallback) when no device exists.
"""

import ctypes
import os
import re

import numpy as np
import pytest

from tests.conftest import ROOT

HEADER = os.path.join(ROOT, "include", "dpp.h")
LIB = os.path.join(ROOT, "paper_1808_08328_b200", "libdpp.so")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(dpp_[a-z0-9_]+)\s*\(", text)) - {"dpp_randn_fn", "dpp_apply_fn"})


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "run __graft_entry__.build() first"
    lib = ctypes.CDLL(LIB)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert len(declared_symbols()) >= 40


def test_binding_covers_every_symbol():
    from paper_1808_08328_b200 import _native
    bound = set(_native.SIGNATURES) | {"dpp_last_error"}
    assert set(declared_symbols()) <= bound


@pytest.mark.parametrize("dim,kind,n", [(2, "tri", 3), (2, "quad", 3), (3, "tet", 2), (3, "hex", 2),
                                        (2, "tri", 7), (3, "tet", 3)])
def test_native_mesh_numbering_matches_reference(golden, dim, kind, n):
    import paper_1808_08328_b200 as dpp
    m = dpp.generate_unit_mesh(dim, kind, n)
    p = f"mesh/{kind}{n}/"
    for a in ("vertices", "cells", "facet_vertex_ids", "cell_facets", "cell_facet_signs",
              "facet_plus", "facet_minus"):
        assert np.array_equal(getattr(m, a), golden[p + a]), a
    J, det = m.jacobians()
    assert np.array_equal(J, golden[p + "J"])
    assert np.array_equal(det, golden[p + "det"])      # numpy's slogdet path, bitwise
    assert np.allclose(m.facet_normals, golden[p + "facet_normals"], rtol=0, atol=1e-15)
    assert np.allclose(m.facet_measures, golden[p + "facet_measures"], rtol=1e-15, atol=0)


@pytest.mark.parametrize("dim,kind,n", [(3, "tet", 12), (2, "tri", 33), (3, "hex", 9)])
def test_native_mesh_matches_oracle_at_larger_sizes(dim, kind, n):
    import oracle
    import paper_1808_08328_b200 as dpp
    m, o = dpp.generate_unit_mesh(dim, kind, n), oracle.generate_unit_mesh(dim, kind, n)
    for a in ("cells", "facet_vertex_ids", "cell_facets", "cell_facet_signs", "facet_plus",
              "facet_minus", "vertices"):
        assert np.array_equal(getattr(m, a), getattr(o, a)), a
    assert np.array_equal(m.jacobians()[1], o.det)


def test_mesh_from_user_arrays_and_errors():
    import paper_1808_08328_b200 as dpp
    m = dpp.Mesh(2, dpp.CellKind.TRI, 1, np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]]),
                 np.array([[0, 1, 2]]))
    assert m.n_facets == 3 and len(m.boundary_facets) == 3
    with pytest.raises(ValueError):
        dpp.generate_unit_mesh(2, "tet", 2)
    with pytest.raises(ValueError):
        dpp.generate_unit_mesh(2, "tri", 0)


def test_option_grammar_mirrors_reference():
    import paper_1808_08328_b200 as dpp
    from paper_1808_08328_b200.blocksolve import flatten
    cfg = dpp.parse_options(dpp.SCALE_SPLIT_OPTIONS)
    assert cfg.split.groups == ((0, 1), (2, 3)) and cfg.split.split_type == "additive"
    assert cfg.split.children[0].split.children[1].pc_type == "amg"
    arr, n = flatten(cfg.split)
    assert n == 3 and arr[0].split_type == 0 and arr[1].split_type == 1
    assert list(arr[0].child_node) == [1, 2] and list(arr[1].child_type) == [0, 1]
    f = dpp.parse_options(dpp.FIELD_SPLIT_OPTIONS)
    arr, n = flatten(f.split)
    assert n == 2 and arr[0].split_type == 1 and list(arr[0].child_type) == [0, 2]
    assert list(arr[1].child_type) == [1, 1]
    with pytest.raises(dpp.OptionError):
        dpp.parse_options(dpp.SCALE_SPLIT_OPTIONS + ["-pc_bogus_option", "1"])
    with pytest.raises(dpp.OptionError):
        dpp.parse_options(["-ksp_type"])
    with pytest.raises(ValueError):
        dpp.method_config("diagonal")
    assert dpp.method_config("field", rtol=1e-9).rtol == 1e-9


def _no_device():
    try:
        import torch
        return not torch.cuda.is_available()
    except Exception:
        return True


@pytest.mark.skipif(not _no_device(), reason="only meaningful without a CUDA device")
def test_compute_paths_fail_loudly_without_device():
    import scipy.sparse as sp

    import paper_1808_08328_b200 as dpp
    with pytest.raises(dpp.DeviceUnavailable):
        dpp.spmv(sp.identity(3, format="csr"), np.ones(3))
    m = dpp.generate_unit_mesh(2, "tri", 2)
    p = dpp.DppParameters()
    with pytest.raises(dpp.DeviceUnavailable):
        dpp.assemble(m, "cgvms", p, dpp.boundary_data(dpp.mms_2d(p), m))


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1808_08328_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
