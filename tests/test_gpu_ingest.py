"""Device ingest (cpfit_from_coords) and .tns parsing vs the reference's own
outputs (tests/golden/ingest.npz): keys bit-exact and duplicate sums
bit-identical to np.add.reduceat's order (segments of 3000 and 100 equal
keys exercise numpy's pairwise recursion and eight-accumulator blocks).
SURVEY 8(f) rank 3."""

import os

import numpy as np
import pytest
import torch

from conftest import golden

import paper_1910_02371_b200 as cp
from paper_1910_02371_b200 import tensor_io
from paper_1910_02371_b200.core import from_coords_device

pytestmark = pytest.mark.gpu


def test_from_coords_duplicates_bit_exact():
    z = golden("ingest")
    shape = tuple(int(d) for d in z["a_shape"])
    t = cp.from_coords([z[f"a_c{q}"] for q in range(3)], z["a_vals"], shape)
    assert np.array_equal(t.keys, z["a_keys"])
    assert np.array_equal(t.values.view(np.uint64), z["a_out"].view(np.uint64))
    # device tensors in, same result; the pattern is usable right away
    tc = from_coords_device([torch.from_numpy(z[f"a_c{q}"]).cuda() for q in range(3)],
                            torch.from_numpy(z["a_vals"]).cuda(), shape)
    assert np.array_equal(tc.keys, z["a_keys"])
    f = [np.random.default_rng(0).standard_normal((d, 3)) for d in shape]
    ref = cp.SparseTensor(shape, z["a_keys"], z["a_out"])
    assert np.allclose(cp.mttkrp(tc, f, 1), cp.mttkrp(ref, f, 1), rtol=1e-13, atol=0)


def test_from_coords_order4_int32():
    z = golden("ingest")
    shape = tuple(int(d) for d in z["b_shape"])
    t = cp.from_coords([z[f"b_c{q}"] for q in range(4)], z["b_vals"], shape)
    assert np.array_equal(t.keys, z["b_keys"])
    assert np.array_equal(t.values, z["b_out"])


def test_from_coords_errors_and_empty():
    with pytest.raises(ValueError, match=r"coordinate out of range \[0, 4\) in mode 1"):
        cp.from_coords([np.array([0, 1]), np.array([3, 4]), np.array([0, 0])],
                       np.ones(2), (2, 4, 1))
    with pytest.raises(ValueError, match="equal length"):
        cp.from_coords([np.array([0, 1]), np.array([0, 1])], np.ones(3), (2, 2))
    t = cp.from_coords([np.zeros(0, np.int64)] * 3, np.zeros(0), (2, 3, 4))
    assert t.nnz == 0 and t.shape == (2, 3, 4)
    # explicit zeros are kept, duplicates that cancel stay as entries
    t = cp.from_coords([np.array([1, 0, 1]), np.array([0, 0, 0])], np.array([2.0, 0.0, -2.0]),
                       (2, 1))
    assert list(t.keys) == [0, 1] and list(t.values) == [0.0, 0.0]


def test_parse_tns_matches_reference(tmp_path):
    z = golden("ingest")
    path = os.path.join(tmp_path, "x.tns")
    with open(path, "w") as fh:
        fh.write(str(z["tns_text"]))
    t = tensor_io.parse_tns(path)
    assert t.shape == tuple(int(d) for d in z["tns_shape"])
    assert np.array_equal(t.keys, z["tns_keys"])
    assert np.array_equal(t.values, z["tns_vals"])
    out = os.path.join(tmp_path, "y.tns")
    tensor_io.write_tns(t, out)
    t2 = tensor_io.parse_tns(out)
    assert np.array_equal(t2.keys, t.keys) and np.array_equal(t2.values, t.values)
