"""CPCompletion (estimator.py) on the GPU vs the reference estimator's own
fit / predict / score (tests/golden/estimator.npz)."""

import numpy as np
import pytest
from sklearn.base import clone

from conftest import golden

import paper_1910_02371_b200 as cp

pytestmark = pytest.mark.gpu


def test_fit_predict_score_match_reference():
    z = golden("estimator")
    m = cp.CPCompletion(rank=2, max_iters=6, seed=3, deterministic=True).fit(z["X"], z["y"])
    for n in range(3):
        assert np.allclose(m.factors_[n], z[f"f{n}"], rtol=1e-9, atol=1e-12)
    assert m.n_iter_ == int(z["n_iter"])
    assert m.objective_ == pytest.approx(float(z["objective"]), rel=1e-10)
    assert np.allclose(m.predict(z["Xq"]), z["pred"], rtol=1e-10, atol=1e-13)
    assert m.score(z["X"], z["y"]) == pytest.approx(float(z["score"]), rel=1e-9)
    c = clone(m)
    assert c.get_params()["rank"] == 2 and not hasattr(c, "factors_")
    with pytest.raises(ValueError, match="expected 3"):
        m.predict(np.zeros((2, 2), dtype=np.int64))
    with pytest.raises(ValueError, match="out of range in mode 0"):
        m.predict(np.array([[99, 0, 0]]))
