"""GPU parity of `sparse_matmul` (csrc/spgemm.cu) against the reference-written fixture and the reference's
own cases (pkg/tests/test_sparse.py:236-266), and `sweep` / `to_json` / `to_csv` end to end
(pkg/tests/test_cli.py:120-175)."""

import csv
import io
import json

import numpy as np
import pytest

from _golden import load

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2303_08881_b200 as pkg
    return pkg


def test_sparse_matmul_bit_exact(P):
    misc = load("misc.npz")
    for name in misc.names("spgemm.names"):
        a, b, c = (misc.csr(f"spgemm.{name}.{k}", P.CsrMatrix) for k in "abc")
        got = P.sparse_matmul(a, b)
        assert got.shape == c.shape, name
        assert np.array_equal(got.row_ptr, c.row_ptr), name
        assert np.array_equal(got.col_idx, c.col_idx), name
        assert np.array_equal(got.values, c.values), name


def test_sparse_matmul_reference_cases(P):
    rng = np.random.default_rng(4)
    d = rng.standard_normal((6, 6))
    d[rng.random((6, 6)) < 0.5] = 0.0
    a = P.csr_from_dense(d)
    assert np.array_equal(P.sparse_matmul(a, P.csr_identity(6)).to_dense(), d)
    sq = P.csr_from_dense(np.array([[1.0, 1.0], [0.0, 1.0]]))
    assert np.array_equal(P.sparse_matmul(sq, sq).to_dense(), [[1.0, 2.0], [0.0, 1.0]])
    z = P.csr_from_coo(2, 2, np.array([], dtype=np.int64), np.array([], dtype=np.int64), np.array([]))
    assert P.sparse_matmul(P.csr_from_dense(np.array([[1.0, 2.0], [3.0, 4.0]])), z).nnz == 0
    p = P.sparse_matmul(P.csr_from_dense(np.ones((2, 2))), P.csr_from_dense(np.array([[1.0, 1.0], [-1.0, -1.0]])))
    assert p.nnz == 4 and np.array_equal(p.to_dense(), np.zeros((2, 2)))      # cancelled entries are kept
    with pytest.raises(ValueError):
        P.sparse_matmul(P.csr_identity(2), P.csr_identity(3))
    # against scipy on a stencil-sized product (values to rounding: scipy sums in another order)
    import scipy.sparse as sp
    g = P.poisson3d(12, 11, 10)
    s = sp.csr_matrix((g.values, g.col_idx, g.row_ptr), shape=g.shape)
    ref = (s @ s).tocsr()
    ref.sort_indices()
    got = P.sparse_matmul(g, g)
    assert np.array_equal(got.row_ptr, ref.indptr) and np.array_equal(got.col_idx, ref.indices)
    assert np.allclose(got.values, ref.data, rtol=1e-14, atol=1e-14)


def _small_cfg(P, **kw):
    return P.RunConfig(problem=P.ProblemSpec("poisson3d", (8, 8, 8)), domains=kw.pop("domains", 2), **kw)


def test_sweep_errors_become_rows_and_order_is_kept(P, tmp_path):
    bad = P.RunConfig(problem=P.ProblemSpec("file", path=str(tmp_path / "no.mtx")))
    records = P.sweep([_small_cfg(P), bad, _small_cfg(P, precond="l1bj")])
    assert len(records) == 3
    assert records[0]["error"] is None and records[0]["converged"]
    assert records[1]["error"].startswith("FileNotFoundError") and records[1]["its"] is None
    assert records[2]["error"] is None and records[2]["precond"] == "l1bj"


def test_sweep_serialisation(P, tmp_path):
    import jsonschema
    bad = P.RunConfig(problem=P.ProblemSpec("file", path=str(tmp_path / "no.mtx")))
    records = P.sweep([_small_cfg(P, history=True), bad])
    doc = json.loads(P.to_json(records))
    jsonschema.validate(doc, json.loads(P.REPORT_SCHEMA))
    rows = list(csv.reader(io.StringIO(P.to_csv(records))))
    assert tuple(rows[0]) == P.COLUMNS
    good = dict(zip(P.COLUMNS, rows[1]))
    assert good["converged"] == "true" and good["error"] == ""
    assert float(good["final_relres"]) == records[0]["final_relres"]
    assert "history" not in P.to_csv(records)


def test_matrix_market_problem_through_the_pipeline(P, tmp_path):
    """A matrix written to disk and read back solves like the generated one (mmio.py + ProblemSpec("file"))."""
    a = P.poisson3d(8, 8, 8)
    path = tmp_path / "p.mtx"
    P.write_matrix_market(path, a, symmetric=True)
    rec_file, _ = P.run(P.RunConfig(problem=P.ProblemSpec("file", path=str(path)), domains=4, precond="schur"))
    assert rec_file["converged"] and rec_file["n"] == 512
