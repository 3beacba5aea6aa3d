"""Host logic of the ctf-style façade: einsum subscripts -> MTTKRP plan
(PAPER.md:120-131 patterns), and rejection of contractions off the path."""

import pytest

from paper_1910_02371_b200.ctf import plan_einsum


def test_mttkrp_patterns():
    assert plan_einsum("ijk,jr,kr->ir", [3, 2, 2]) == (0, "r", [[], [1], [2]])
    assert plan_einsum("ijk,ir,kr->jr", [3, 2, 2]) == (1, "r", [[1], [], [2]])
    assert plan_einsum("ijk,ir,jr->kr", [3, 2, 2]) == (2, "r", [[1], [2], []])
    assert plan_einsum("ijkl,ir,jr,lr->kr", [4, 2, 2, 2]) == (2, "r", [[1], [2], [], [3]])
    # CCD++ numerator and denominator (repeated vectors on a mode)
    assert plan_einsum("ijk,j,k->i", [3, 1, 1]) == (0, None, [[], [1], [2]])
    assert plan_einsum("ijk,j,j,k,k->i", [3, 1, 1, 1, 1]) == (0, None, [[], [1, 2], [3, 4]])
    assert plan_einsum("ij,jr->ir", [2, 2]) == (0, "r", [[], [1]])


@pytest.mark.parametrize("spec,nd", [
    ("ir,jr,kr->ijk", [2, 2, 2]),          # dense reconstruction: not this path
    ("ijk,jr,kr->i", [3, 2, 2]),           # rank index summed away
    ("ijk,jr->ir", [3, 2]),                # mode k not contracted
    ("ijk,jr,kr,ir->ir", [3, 2, 2, 2]),    # output mode contracted
    ("ijk,jr,ks->ir", [3, 2, 2]),          # two rank indices
    ("ijk,rj,kr->ir", [3, 2, 2]),          # factor not (mode, rank)
    ("ijk,jr,kr->ri", [3, 2, 2]),          # output not (mode, rank)
    ("iik,ir->kr", [3, 2]),                # repeated tensor index
    ("ijk,jr,kr", [3, 2, 2]),              # implicit output
    ("ijk,jr,kr->ir", [3, 2]),             # operand count
])
def test_rejects_contractions_off_the_path(spec, nd):
    with pytest.raises(ValueError):
        plan_einsum(spec, nd)
