"""CPU-side checks: the C-ABI library loads and exports every symbol the header
declares, the ctypes table matches the header, and the host logic of the
reference-facing API (validation, parsing, configuration errors) behaves like
the reference.  No kernel is launched here."""

import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_text(name="ddilu_b200.h"):
    text = open(os.path.join(ROOT, "include", name)).read()
    return re.sub(r"/\*.*?\*/", "", text, flags=re.S)


def _header_symbols(name="ddilu_b200.h"):
    return sorted(set(re.findall(r"\b(ddilu_[a-z0-9_]+)\s*\(", _header_text(name))))


def test_library_exports_every_declared_symbol():
    from paper_2303_08881_b200 import _lib
    lib = _lib.load()
    names = _header_symbols()
    assert len(names) >= 40
    for name in names:
        assert hasattr(lib, name), f"{name} declared in include/ddilu_b200.h but not exported"
    assert sorted(_lib.SIGNATURES) == names, "ctypes table and header disagree"


def test_experiment_entries_are_not_part_of_the_product_abi():
    """Alternative kernels, tuning knobs and diagnostics live in ddilu_b200_experiments.h; a product build
    exports none of them, an experiments build (DDILU_EXPERIMENTS=1) exports all of them."""
    from paper_2303_08881_b200 import _lib
    lib = _lib.load()
    names = _header_symbols("ddilu_b200_experiments.h")
    assert sorted(_lib.EXPERIMENT_SIGNATURES) == names, "ctypes table and experiments header disagree"
    assert not set(names) & set(_header_symbols())
    present = [hasattr(lib, n) for n in names]
    assert all(present) if _lib.has_experiments() else not any(present)


def test_header_argument_counts_match_ctypes_table():
    from paper_2303_08881_b200 import _lib
    for header, table in (("ddilu_b200.h", _lib.SIGNATURES), ("ddilu_b200_experiments.h", _lib.EXPERIMENT_SIGNATURES)):
        for name, args in re.findall(r"\b(ddilu_[a-z0-9_]+)\s*\(([^)]*)\)\s*;", _header_text(header)):
            nargs = 0 if args.strip() in ("", "void") else len(args.split(","))
            assert nargs == len(table[name][1]), name


def test_no_cpu_fallback_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    import paper_2303_08881_b200 as P
    from paper_2303_08881_b200._lib import DdiluError
    a = P.poisson2d(4, 4)
    with pytest.raises(DdiluError):
        P.spmv(a, np.ones(16))
    with pytest.raises(DdiluError):
        P.ilu0(a)


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2303_08881_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "oracle" not in src.replace("test-oracle", ""), fn


def test_fill_rule_and_configs():
    """tests/test_factor.py:38-60, tests/test_krylov.py config validation."""
    import paper_2303_08881_b200 as P
    for text in ("ilu0", "iluk:2", "ilut:0.01,10"):
        assert str(P.FillRule.parse(text)) == text
    r = P.FillRule.parse("ilut:0.5,7")
    assert r.kind == "ilut" and r.tau == 0.5 and r.maxfill == 7
    for bad in ("iluk", "ilut:0.1", "bogus", "ilu0:1"):
        with pytest.raises(ValueError):
            P.FillRule.parse(bad)
    with pytest.raises(ValueError):
        P.FillRule("ilut", tau=0.1, maxfill=0)
    with pytest.raises(ValueError):
        P.KrylovConfig(restart=0)
    with pytest.raises(ValueError):
        P.KrylovConfig(rtol=0.0)
    with pytest.raises(ValueError):
        P.RunConfig(P.ProblemSpec("poisson2d", (4, 4)), precond="nope")
    with pytest.raises(ValueError):
        P.ProblemSpec("poisson3d", (4, 4))


def test_csr_validation_and_permutation():
    """sparse.py:87-112, 168-212 semantics."""
    import paper_2303_08881_b200 as P
    ok = P.csr_from_arrays(2, 2, [0, 1, 2], [0, 1], [1.0, 2.0])
    assert ok.nnz == 2 and ok.shape == (2, 2)
    with pytest.raises(ValueError):
        P.csr_from_arrays(2, 2, [0, 2, 2], [1, 0], [1.0, 2.0])      # not increasing
    with pytest.raises(ValueError):
        P.csr_from_arrays(2, 2, [0, 1, 2], [0, 5], [1.0, 2.0])      # out of range
    with pytest.raises(ValueError):
        P.csr_from_arrays(2, 2, [0, 1], [0], [1.0])                 # row_ptr length
    P.csr_from_arrays(3, 3, [0, 2, 3, 4], [1, 2, 0, 0], [1.0, 1.0, 1.0, 1.0])  # drop at a row boundary is fine
    with pytest.raises(ValueError):
        P.csr_from_coo(2, 2, [0, 0], [1, 1], [1.0, 2.0])            # duplicate
    perm = P.Permutation.from_order([2, 0, 1])
    assert np.array_equal(perm.forward, [1, 2, 0]) and np.array_equal(perm.inverse, [2, 0, 1])
    with pytest.raises(ValueError):
        P.Permutation([0, 0, 1])
    d = np.array([[1.0, 0.0], [2.0, 3.0]])
    assert np.array_equal(P.csr_from_dense(d).to_dense(), d)


def test_generators_match_reference_fixtures(golden_pipeline):
    import paper_2303_08881_b200 as P
    from _golden import same_csr
    g = golden_pipeline
    same_csr(P.aniso2d(16, 16, (1.0, 0.01)), g, "p.aniso2d_16.a")
    same_csr(P.aniso3d(10, 10, 10, (1.0, 1.0, 0.01)), g, "p.aniso3d_10.a")
    same_csr(P.poisson3d(9, 8, 7), g, "p.poisson3d_9x8x7.a")
    same_csr(P.convdiff3d(8, 8, 8, (20.0, -10.0, 5.0)), g, "p.convdiff3d_8.a")
    same_csr(P.convdiff27(8, 8, 8, (10.0, 10.0, 10.0)), g, "p.cd27_8.a")


def test_box_factors_and_row_blocks():
    """tests/test_ordering.py partition maps: factor placement and near-equal row blocks."""
    from paper_2303_08881_b200.ordering import _box_factors, row_block_owner
    assert _box_factors((256, 256, 256), 8) == [2, 2, 2]
    assert _box_factors((128, 128, 128), 4) == [2, 2, 1]
    assert _box_factors((128, 128, 128), 2) == [2, 1, 1]
    assert _box_factors((9, 7), 3) == [3, 1]
    assert np.array_equal(row_block_owner(7, 3), [0, 0, 0, 1, 1, 2, 2])
    with pytest.raises(ValueError):
        row_block_owner(2, 3)
