"""The pairwise (hypersparse) baseline on the device vs the reference's own
outputs (tests/golden/hypersparse.npz): CCSR structure bit-exact, values
bit-exact where the reference's summation order is reproduced (COO build,
matricize, sums, canonical butterfly, CCSR x dense, TTM, pairwise TTTP,
pairwise MTTKRP), 1e-13 for the eager butterfly.  SURVEY 8(f) rank 4."""

import numpy as np
import pytest

from conftest import golden

import paper_1910_02371_b200 as cp
from paper_1910_02371_b200 import hypersparse as H

pytestmark = pytest.mark.gpu


def ccsr(z, tag):
    gr, gc = (int(x) for x in z[f"{tag}_shape"])
    return H.CcsrMatrix(gr, gc, z[f"{tag}_rows"], z[f"{tag}_offs"], z[f"{tag}_cols"],
                        z[f"{tag}_vals"])


def same(a, z, tag, exact=True):
    assert (a.global_rows, a.global_cols) == tuple(int(x) for x in z[f"{tag}_shape"])
    assert np.array_equal(a.nnz_row_ids, z[f"{tag}_rows"])
    assert np.array_equal(a.row_offsets, z[f"{tag}_offs"])
    assert np.array_equal(a.col_ids, z[f"{tag}_cols"])
    if exact:
        assert np.array_equal(a.values.view(np.uint64), z[f"{tag}_vals"].view(np.uint64))
    else:
        assert np.allclose(a.values, z[f"{tag}_vals"], rtol=1e-13, atol=1e-13)


def tensor(z, p=""):
    return cp.SparseTensor(tuple(int(d) for d in z[f"{p}dims"]), z[f"{p}keys"], z[f"{p}vals"])


def test_coo_matricize_spmm_sum():
    z = golden("hypersparse")
    a = H.ccsr_from_coo(z["coo_r"], z["coo_c"], z["coo_v"], 100_000, 300)
    same(a, z, "coo")
    t = tensor(z, "t_")
    for tag, rm, cm in (("mat_native", (0, 1), (2, 3)), ("mat_perm", (3, 1), (0, 2)),
                        ("mat_rowsonly", (2, 0, 3, 1), ())):
        same(H.matricize_to_ccsr(t, rm, cm), z, tag)
    p = H.ccsr_times_dense(a, z["spmm_b"])
    assert np.array_equal(p.fiber_keys, z["spmm_keys"])
    assert np.array_equal(p.payload, z["spmm_payload"])
    same(H.ccsr_sum(a, ccsr(z, "a2")), z, "sum12")
    same(H.ccsr_sum(a, ccsr(z, "a3")), z, "sum13")
    with pytest.raises(ValueError):
        H.matricize_to_ccsr(t, (0, 1), (1, 2))
    with pytest.raises(ValueError, match="dimension mismatch"):
        H.ccsr_times_dense(a, np.ones((7, 2)))


@pytest.mark.parametrize("k", [2, 3])
@pytest.mark.parametrize("canonical", [True, False])
def test_butterfly_reduce_scatter(k, canonical):
    z = golden("hypersparse")
    parts = [ccsr(z, f"bf_in{p}") for p in range(5)]
    shards = H.butterfly_reduce_scatter(parts, k=k, canonical=canonical)
    tag = f"bf_k{k}_c{int(canonical)}"
    for p, sh in enumerate(shards):
        same(sh, z, f"{tag}_s{p}", exact=canonical)
    same(H.butterfly_gather(shards), z, f"{tag}_all", exact=canonical)


def test_ttm_and_pairwise_kernels():
    z = golden("hypersparse")
    t = tensor(z, "t_")
    zz = H.ttm(t, z["ttm_w"], 2)
    assert np.array_equal(zz.fiber_keys, z["ttm_keys"])
    assert np.array_equal(zz.payload, z["ttm_payload"])
    f4 = [z[f"pw_f{n}"] for n in range(4)]
    for mode in range(4):
        assert np.array_equal(H.pairwise_mttkrp(t, f4, mode), z[f"pw_mttkrp{mode}"])
    t3 = tensor(z, "t3_")
    for R in (1, 7, 8, 20):
        fs = [z[f"pt{R}_f{n}"] for n in range(3)]
        assert np.array_equal(H.pairwise_tttp(t3, fs).values, z[f"pt{R}_out"])
        assert np.array_equal(H.pairwise_tttp(t3, [None, fs[1], fs[2]]).values,
                              z[f"pt{R}_none_out"])
        assert np.array_equal(H.pairwise_mttkrp(t3, fs, 1), z[f"pt{R}_mttkrp1"])
        # the all-at-once kernels agree to rounding
        assert np.allclose(cp.mttkrp(t3, fs, 1), z[f"pt{R}_mttkrp1"], rtol=1e-12, atol=1e-12)
