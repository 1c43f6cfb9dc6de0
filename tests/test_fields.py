"""Discrete fields, L2 errors and the run_case harness (reference assembly.py:591-644,
spectrum.py:88-276), pinned to the unmodified reference (tests/golden/fields.npz,
run_case.json, run_case_*.csv from tests/golden/make_golden_fields.py).

CPU: the oracle's restatement against the golden values; the CSV schema / reader on the
reference-written files.  GPU: DiscreteField.evaluate_all, l2_error (device manufactured
solution and host-callable exact fields) and spectrum.run_case of this package.
"""

import json
import os

import numpy as np
import pytest

from tests.conftest import GOLDEN

CASES = [("hdiv", 2, "tri", 6), ("hdiv", 2, "quad", 5), ("hdiv", 3, "tet", 3), ("hdiv", 3, "hex", 3),
         ("cgvms", 2, "tri", 6), ("cgvms", 2, "quad", 5), ("cgvms", 3, "tet", 3), ("cgvms", 3, "hex", 3),
         ("dgvms", 2, "tri", 4), ("dgvms", 3, "tet", 2)]
REF_PTS = {2: np.array([[0.2, 0.3], [0.1, 0.1], [0.25, 0.5]]),
           3: np.array([[0.2, 0.3, 0.1], [0.1, 0.1, 0.1], [0.25, 0.2, 0.3]])}
FIELDS = ("u1", "p1", "u2", "p2")


@pytest.fixture(scope="module")
def gf():
    with np.load(os.path.join(GOLDEN, "fields.npz")) as z:
        return {k: z[k] for k in z.files}


def _split(x, sizes):
    out, s = {}, 0
    for name, n in zip(FIELDS, sizes):
        out[name] = x[s:s + n]
        s += n
    return out


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-{c[2]}{c[3]}")
def test_oracle_fields_match_reference(case, gf):
    import oracle
    from oracle import fields as of
    form, dim, kind, n = case
    p = f"{form}/{kind}{n}/"
    op = oracle.Params(gamma_b=(0.0,) * dim)
    m = oracle.generate_unit_mesh(dim, kind, n)
    obs = oracle.assemble(m, form, op, oracle.boundary_data(oracle.mms(dim, op), m))
    x = gf[p + "x"]
    parts = _split(x, [len(obs.rhs[f]) for f in FIELDS])
    for name in FIELDS:
        v = of.evaluate_all(m, form, name, parts[name], REF_PTS[dim])
        ref = gf[p + "eval/" + name]
        assert np.abs(v - ref).max() <= 1e-13 * max(1.0, np.abs(ref).max())
    errs = of.field_errors(obs, x, oracle.mms(dim, op))
    np.testing.assert_allclose([errs[f] for f in FIELDS], gf[p + "l2"], rtol=1e-12)


def test_csv_schema_matches_reference_files():
    from paper_1808_08328_b200 import spectrum
    for name in ("run_case_cgvms_tri8.csv", "run_case_hdiv_tri8.csv"):
        rows = spectrum.read_csv(os.path.join(GOLDEN, name))   # raises on a schema mismatch
        assert len(rows) == 1 and rows[0]["formulation"] in ("cgvms", "hdiv")
    with open(os.path.join(GOLDEN, "run_case_cgvms_tri8.csv")) as fh:
        assert fh.readline().strip().split(",") == list(spectrum.CSV_COLUMNS)


def test_csv_roundtrip_and_digits(tmp_path):
    from paper_1808_08328_b200 import spectrum
    rec = spectrum.SpectrumRecord("cgvms", "tri", 8, 1000, 12, 0.5, 1.5, 2.0,
                                  {"u1": 1e-2, "p1": 1e-3, "u2": 2e-2, "p2": 5e-3})
    path = tmp_path / "s.csv"
    spectrum.write_csv([rec], path)
    row = spectrum.read_csv(path)[0]
    assert float(row["doa_p1"]) == pytest.approx(3.0) and float(row["dos"]) == pytest.approx(-3.0)
    assert float(row["dof_per_s_total"]) == pytest.approx(500.0)
    with pytest.raises(ValueError):
        spectrum.doa(0.0)


# ----------------------------------------------------------------------------- device

@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-{c[2]}{c[3]}")
def test_device_fields_match_reference(case, gf):
    import paper_1808_08328_b200 as dpp
    form, dim, kind, n = case
    p = f"{form}/{kind}{n}/"
    params = dpp.DppParameters(gamma_b=(0.0,) * dim)
    mms = dpp.manufactured_solution(dim, params)
    m = dpp.generate_unit_mesh(dim, kind, n)
    bs = dpp.assemble(m, form, params, dpp.boundary_data(mms, m))
    x = gf[p + "x"]
    fields = dpp.solution_fields(bs, x)
    for name in FIELDS:
        assert isinstance(fields[name], dpp.DiscreteField)
        v = fields[name].evaluate_all(REF_PTS[dim])
        ref = gf[p + "eval/" + name]
        assert v.shape == ref.shape
        assert np.abs(v - ref).max() <= 1e-13 * max(1.0, np.abs(ref).max())
    # device-evaluated manufactured solution
    errs = dpp.field_errors(bs, x, mms)
    np.testing.assert_allclose([errs[f] for f in FIELDS], gf[p + "l2"], rtol=1e-12)
    # host callables (no device tag): evaluated at the device-computed quadrature points
    for name in FIELDS:
        fn = mms.field(name)
        plain = lambda pts, fn=fn: fn(pts)   # noqa: E731
        e = dpp.l2_error(fields[name], plain, m)
        assert e == pytest.approx(errs[name], rel=1e-12)


@pytest.mark.gpu
def test_run_case_matches_reference_harness():
    """This package's spectrum.run_case against the reference's own run_case records."""
    import paper_1808_08328_b200 as dpp
    with open(os.path.join(GOLDEN, "run_case.json")) as fh:
        ref = json.load(fh)
    for key, g in ref.items():
        form, cell, meth = key.split("/")
        kind, n = cell[:-1], int(cell[-1])
        rec = dpp.run_case(form, kind, n, method=meth, rtol=1e-8)
        assert rec.dof == g["dof"] and abs(rec.ksp - g["ksp"]) <= 2
        for f in FIELDS:
            assert rec.l2[f] == pytest.approx(g["l2"][f], rel=1e-7)
        assert rec.dos == pytest.approx(g["dos"])
        assert rec.csv_row()[:4] == [form, kind, str(n), str(g["dof"])]
