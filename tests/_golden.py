"""Helpers to read the reference-generated fixtures in tests/golden/."""

import json
import os

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


class Golden:
    def __init__(self, path):
        with np.load(path, allow_pickle=False) as z:
            self.data = {k: z[k] for k in z.files}

    def __getitem__(self, key):
        return self.data[key]

    def __contains__(self, key):
        return key in self.data

    def csr(self, key, ctor):
        """ctor(n_rows, n_cols, row_ptr, col_idx, values) -> matrix object."""
        sh = self.data[key + ".shape"]
        return ctor(int(sh[0]), int(sh[1]), self.data[key + ".row_ptr"], self.data[key + ".col_idx"],
                    self.data[key + ".values"])

    def names(self, key):
        return [str(s) for s in self.data[key]]


def load(name):
    return Golden(os.path.join(GOLDEN_DIR, name))


def iterations():
    with open(os.path.join(GOLDEN_DIR, "iterations.json")) as fh:
        return json.load(fh)["runs"]


def same_csr(m, g, key, values="exact", rtol=0.0):
    """Compare matrix m (attributes n_rows, n_cols, row_ptr, col_idx, values)
    with the fixture under ``key``: pattern bit-exact, values exact or rtol."""
    sh = g[key + ".shape"]
    assert (m.n_rows, m.n_cols) == (int(sh[0]), int(sh[1])), key
    assert np.array_equal(np.asarray(m.row_ptr, dtype=np.int64), g[key + ".row_ptr"]), key + " row_ptr"
    assert np.array_equal(np.asarray(m.col_idx, dtype=np.int64), g[key + ".col_idx"]), key + " col_idx"
    ref = g[key + ".values"]
    got = np.asarray(m.values)
    if values == "exact":
        assert np.array_equal(got, ref), f"{key} values differ (max {np.max(np.abs(got - ref)) if len(ref) else 0})"
    else:
        scale = np.maximum(np.abs(ref), 1e-300)
        assert np.all(np.abs(got - ref) <= rtol * scale + 1e-300), \
            f"{key} values rel err {np.max(np.abs(got - ref) / scale)}"
