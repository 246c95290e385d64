"""Oracle restatement of `sparse_matmul` pinned to the reference-written fixture tests/golden/misc.npz
(generator: tests/golden/make_golden_misc.py), and the host-side Matrix Market reader / writer against the
reference's own test cases (pkg/tests/test_mmio.py).  CPU only."""

import numpy as np
import pytest

from _golden import load


@pytest.fixture(scope="module")
def misc():
    return load("misc.npz")


def test_oracle_sparse_matmul_against_reference(misc):
    from oracle import ddilu_oracle as orc
    for name in misc.names("spgemm.names"):
        a, b, c = (misc.csr(f"spgemm.{name}.{k}", orc.Csr) for k in "abc")
        got = orc.sparse_matmul(a, b)
        assert (got.n_rows, got.n_cols) == (c.n_rows, c.n_cols), name
        assert np.array_equal(got.row_ptr, c.row_ptr), name
        assert np.array_equal(got.col_idx, c.col_idx), name
        assert np.array_equal(got.values, c.values), name
    with pytest.raises(ValueError):
        a = misc.csr("spgemm.rect.a", orc.Csr)
        orc.sparse_matmul(a, a)


# ---- Matrix Market IO (mmio.py:21-73; cases of the reference's pkg/tests/test_mmio.py)


@pytest.fixture(scope="module")
def P():
    import paper_2303_08881_b200 as pkg
    return pkg


def test_mmio_roundtrip_general(P, tmp_path):
    rng = np.random.default_rng(0)
    d = rng.standard_normal((7, 5))
    d[rng.random((7, 5)) < 0.5] = 0.0
    a = P.csr_from_dense(d)
    path = tmp_path / "general.mtx"
    P.write_matrix_market(path, a)
    b = P.read_matrix_market(path)
    assert b.shape == a.shape
    assert np.array_equal(b.to_dense(), d)          # 17 significant digits: exact round trip


def test_mmio_roundtrip_symmetric_expands_triangle(P, tmp_path):
    rng = np.random.default_rng(1)
    d = rng.standard_normal((6, 6))
    d = d + d.T
    d[np.abs(d) < 0.8] = 0.0
    d = (d + d.T) / 2.0
    a = P.csr_from_dense(d)
    path = tmp_path / "sym.mtx"
    P.write_matrix_market(path, a, symmetric=True)
    assert "symmetric" in path.read_text().splitlines()[0]
    assert np.array_equal(P.read_matrix_market(path).to_dense(), d)
    n_diag = int(np.count_nonzero(np.diag(d)))
    stored = sum(1 for line in path.read_text().splitlines() if line and not line.startswith("%")) - 1
    assert a.nnz == 2 * (stored - n_diag) + n_diag


def test_mmio_one_based_and_errors(P, tmp_path):
    path = tmp_path / "one.mtx"
    path.write_text("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 3.5\n")
    assert np.array_equal(P.read_matrix_market(path).to_dense(), [[0.0, 3.5], [0.0, 0.0]])
    with pytest.raises(FileNotFoundError):
        P.read_matrix_market(tmp_path / "absent.mtx")
    bad = {
        "bad.mtx": "not a matrix market file\n1 1 1\n1 1 1.0\n",
        "cplx.mtx": "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1.0 0.0\n",
        "arr.mtx": "%%MatrixMarket matrix array real general\n2 1\n1.0\n2.0\n",
        "skew.mtx": "%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n2 1 1.0\n",
        "oob.mtx": "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n",
    }
    for name, text in bad.items():
        p = tmp_path / name
        p.write_text(text)
        with pytest.raises(ValueError):
            P.read_matrix_market(p)
    with pytest.raises(ValueError):
        P.write_matrix_market("/dev/null", P.csr_from_dense(np.array([[1.0, 2.0], [0.0, 1.0]])), symmetric=True)


def test_serialisation_of_records(P):
    """to_json / to_csv (bench.py:143-195) on hand-made records: fixed columns, true/false, repr floats, empty
    cells for missing values, the history never in the CSV, the JSON valid against REPORT_SCHEMA."""
    import csv
    import io
    import json
    import jsonschema
    good = {"problem": "aniso3d-8x8x8", "n": 512, "p": 8, "precond": "schur", "fill": "ilu0", "its": 12,
            "converged": True, "setup_s": 0.25, "solve_s": 0.125, "final_relres": 7.691622412144931e-09,
            "error": None, "history": [1.0, 0.5]}
    bad = dict.fromkeys(P.COLUMNS)
    bad.update(problem="file", p=1, precond="bj", fill="ilu0", error="FileNotFoundError: no such file")
    rows = list(csv.reader(io.StringIO(P.to_csv([good, bad]))))
    assert tuple(rows[0]) == P.COLUMNS
    g = dict(zip(P.COLUMNS, rows[1]))
    assert g["converged"] == "true" and g["error"] == "" and float(g["final_relres"]) == good["final_relres"]
    e = dict(zip(P.COLUMNS, rows[2]))
    assert e["its"] == "" and e["error"].startswith("FileNotFoundError")
    assert "history" not in P.to_csv([good])
    text = P.to_json([good, bad])
    assert text.endswith("\n")
    doc = json.loads(text)
    assert set(doc) == {"runs"}
    schema = json.loads(P.REPORT_SCHEMA)
    jsonschema.validate(doc, schema)
    jsonschema.validate({"runs": []}, schema)
    with pytest.raises(jsonschema.ValidationError):
        jsonschema.validate({"runs": [{"problem": "x"}]}, schema)
    with pytest.raises(ValueError):
        P.sweep([])
