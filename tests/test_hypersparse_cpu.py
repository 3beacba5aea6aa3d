"""CCSR host logic without a GPU: invariants, restrict_rows, row blocks,
butterfly edge cases (hypersparse.py:23-90, 253-374)."""

import numpy as np
import pytest

from paper_1910_02371_b200 import hypersparse as H


def test_invariants_checked():
    with pytest.raises(ValueError):
        H.CcsrMatrix(2, 2, [0, 0], [0, 1, 2], [0, 1], [1.0, 2.0])
    with pytest.raises(ValueError):
        H.CcsrMatrix(2, 2, [0], [0, 2], [1, 1], [1.0, 2.0])
    a = H.CcsrMatrix(3, 4, [0, 2], [0, 2, 3], [1, 3, 0], [1.0, 2.0, 3.0])
    assert a.nnz == 3 and a.n_nonzero_rows == 2
    d = a.to_dense()
    assert d[0, 1] == 1.0 and d[0, 3] == 2.0 and d[2, 0] == 3.0 and d.sum() == 6.0


def test_restrict_rows_and_blocks():
    a = H.CcsrMatrix(10, 3, [1, 4, 8], [0, 1, 3, 4], [0, 1, 2, 0], [1.0, 2.0, 3.0, 4.0])
    r = H.restrict_rows(a, 2, 9)
    assert r.nnz_row_ids.tolist() == [4, 8] and r.row_offsets.tolist() == [0, 2, 3]
    assert H.restrict_rows(a, 5, 8).nnz == 0
    assert H.row_block_bounds(10, 3) == [0, 4, 8, 10]
    assert H.row_block_bounds(2, 4) == [0, 1, 2, 2, 2]


def test_butterfly_edge_cases():
    e = H.ccsr_empty(4, 4)
    with pytest.raises(ValueError):
        H.butterfly_reduce_scatter([])
    with pytest.raises(ValueError):
        H.butterfly_reduce_scatter([e, e], k=1)
    with pytest.raises(ValueError):
        H.butterfly_reduce_scatter([e, H.ccsr_empty(4, 5)])
    assert H.butterfly_reduce_scatter([e]) == [e]
    with pytest.raises(ValueError):
        H.butterfly_gather([e, e])
