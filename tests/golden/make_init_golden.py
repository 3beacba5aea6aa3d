"""Golden vectors for the initialisation laws, from the REFERENCE package:
``init_state`` with init = uniform / gaussian / svd (rank below and above what
the unfoldings can supply), ``calibrate_init`` and the synthetic generators.
Writes tests/golden/init_state.npz.  Run here (needs /root/reference):
    python tests/golden/make_init_golden.py"""
import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.path.insert(0, "/root/reference/pkg/src")
import cpfit  # noqa: E402
from cpfit import optim as ro  # noqa: E402

out = {}
t, truth = cpfit.gen_low_rank((14, 9, 11), 3, 0.4, "gaussian", cpfit.RngState(21).child(2))
out["keys"], out["values"], out["shape"] = t.keys, t.values, np.array(t.shape)
for k, f in enumerate(truth):
    out[f"truth{k}"] = f
cases = [("uniform", 6, False), ("gaussian", 6, False), ("svd", 4, False), ("svd", 12, False),
         ("uniform", 5, True), ("gaussian", 5, True)]
for init, rank, calib in cases:
    cfg = ro.SolverConfig(rank=rank, init=init, seed=13, calibrate_init=calib)
    st = ro.init_state(t, cfg)
    for k, f in enumerate(st.factors):
        out[f"{init}_{rank}_{int(calib)}_{k}"] = f
ft = cpfit.gen_function_tensor((7, 8, 5), 0.5, cpfit.RngState(4))
out["func_keys"], out["func_values"] = ft.keys, ft.values
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "init_state.npz")
np.savez_compressed(path, **out)
print(path, len(out), "arrays")
