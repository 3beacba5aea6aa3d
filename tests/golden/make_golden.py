"""Generate golden vectors by running the REFERENCE package (cpfit) itself.

Run here, in the build container, where /root/reference exists:

    python tests/golden/make_golden.py

It imports ``cpfit`` read-only from /root/reference/pkg/src (numba JIT on,
cache in /tmp), builds seeded inputs, runs the reference's own public API and
writes compressed ``.npz`` fixtures next to this script.  The fixtures travel
to the GPU box; /root/reference does not, so nothing else reads it at run time.

Fixtures:
  kernels_small.npz  -- 120 random small cases (order 2-4, dims <= 6, R <= 4):
                        tttp (with absent factors), mttkrp, gram_blocks,
                        solve_factor, counting_sort_by_mode
  layout.npz         -- from_coords with duplicates, counting sort perms of a
                        20k-entry tensor, linearize/delinearize round trip
  philox.npz         -- RngState draws and SparseTensor.sample keep-sets
  cfg1.npz           -- BASELINE cfg 1: tttp, mttkrp x3, 5 ALS sweeps (+rmse),
                        2 CCD++ sweeps, 3 SGD steps, all from the reference
  drivers_small.npz  -- ALS/CCD/SGD single sweeps and run() traces, small case
  generalized.npz    -- Poisson log-link (and generalized least squares):
                        derivative tensors / objective incl. exp clamp counts,
                        inner-Newton ALS and CCD++ sweeps, SGD steps, run()
                        traces
  ingest.npz         -- from_coords with heavy duplicates (segments < 8,
                        8..128 and > 128 long: numpy's reduceat/pairwise
                        order), order-4 int32 coordinates, and parse_tns of a
                        generated .tns text
  hypersparse.npz    -- the pairwise baseline: ccsr_from_coo, matricize
                        (native and permuted modes), ccsr_times_dense,
                        ccsr_sum with cancellations, butterfly reduce-scatter
                        (canonical and eager, k = 2 / 3, P = 5), ttm,
                        pairwise_mttkrp (orders 3 / 4), pairwise_tttp (R up
                        to 20, absent factors)
  cli.npz            -- `cpfit gen` output bytes and `cpfit run --deterministic`
                        trace CSVs (als / ccd / sgd / gn, ls and poisson)
  second_order.npz   -- hessian_matvec (ls/poisson x gauss_newton/newton),
                        gradient_blocks, gn_step trajectories (ls GN, ls
                        Newton, poisson GN) and run(algorithm=gn/newton) traces
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.path.insert(0, "/root/reference/pkg/src")

import cpfit  # noqa: E402  (the reference)
from cpfit import kernels as rk  # noqa: E402
from cpfit import optim as ro  # noqa: E402

from paper_1910_02371_b200 import synth  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def random_sparse(shape, density, rng, ensure_nonempty=True):
    total = int(np.prod(shape))
    mask = rng.random(total) < density
    if ensure_nonempty and not mask.any():
        mask[rng.integers(0, total)] = True
    keys = np.flatnonzero(mask).astype(np.uint64)
    values = rng.standard_normal(keys.size)
    return cpfit.SparseTensor(shape, keys, values)


def kernels_small():
    rng = np.random.default_rng(20240)
    out = {}
    n_cases = 120
    for c in range(n_cases):
        order = int(rng.integers(2, 5))
        dims = tuple(int(d) for d in rng.integers(1, 7, order))
        rank = int(rng.integers(1, 5))
        t = random_sparse(dims, 0.45, rng, ensure_nonempty=(c % 7 != 0))
        factors = [rng.standard_normal((d, rank)) for d in dims]
        mode = int(rng.integers(0, order))
        absent = -1
        if order > 2 and rng.random() < 0.4:
            absent = int(rng.integers(0, order))
        tf = list(factors)
        if absent >= 0:
            tf[absent] = None
        weights = t.with_values(np.abs(t.values) + 0.1)
        rhs = rng.standard_normal((dims[mode], rank))
        reg = float(rng.random() * 0.5 + 0.1)
        p = f"c{c}_"
        out[p + "dims"] = np.array(dims, dtype=np.int64)
        out[p + "keys"] = t.keys
        out[p + "values"] = t.values
        out[p + "mode"] = np.array(mode)
        out[p + "absent"] = np.array(absent)
        out[p + "reg"] = np.array(reg)
        out[p + "rhs"] = rhs
        for n, f in enumerate(factors):
            out[p + f"f{n}"] = f
        out[p + "tttp"] = rk.tttp(t, tf).values
        out[p + "mttkrp"] = rk.mttkrp(t, factors, mode)
        out[p + "gram"] = rk.gram_blocks(weights, factors, mode)
        out[p + "solve"] = rk.solve_factor(weights, factors, rhs, mode, reg=reg)
        perm, offsets = cpfit.counting_sort_by_mode(t, mode)
        out[p + "perm"] = perm
        out[p + "offsets"] = offsets
    out["n_cases"] = np.array(n_cases)
    np.savez_compressed(os.path.join(HERE, "kernels_small.npz"), **out)


def layout():
    rng = np.random.default_rng(77)
    out = {}
    dims = (7, 3, 9, 2)
    coords = [rng.integers(0, d, 300) for d in dims]
    vals = rng.standard_normal(300)
    t = cpfit.from_coords(coords, vals, dims)
    out["fc_dims"] = np.array(dims, dtype=np.int64)
    out["fc_coords"] = np.stack(coords).astype(np.int64)
    out["fc_values_in"] = vals
    out["fc_keys"] = t.keys
    out["fc_values"] = t.values
    dims2 = (50, 40, 30)
    t2 = random_sparse(dims2, 20_000 / 60_000, rng)
    out["cs_dims"] = np.array(dims2, dtype=np.int64)
    out["cs_keys"] = t2.keys
    for mode in range(3):
        perm, offsets = cpfit.counting_sort_by_mode(t2, mode)
        out[f"cs_perm{mode}"] = perm
        out[f"cs_offsets{mode}"] = offsets
    dims3 = (480_189, 17_770, 2_182)
    keys3 = np.sort(rng.integers(0, int(np.prod(np.array(dims3, dtype=object))), 5000,
                                 dtype=np.uint64))
    out["dl_dims"] = np.array(dims3, dtype=np.int64)
    out["dl_keys"] = keys3
    out["dl_coords"] = np.stack(cpfit.delinearize_many(keys3, dims3))
    np.savez_compressed(os.path.join(HERE, "layout.npz"), **out)


def philox():
    out = {}
    cases = [(0, ()), (42, (1,)), (123, (1, 7)), (5, (1, 3)), (2**40 + 3, (0,))]
    for i, (seed, path) in enumerate(cases):
        g = cpfit.RngState(seed, path).generator()
        out[f"u{i}_seed"] = np.array(seed, dtype=np.uint64)
        out[f"u{i}_path"] = np.array(path, dtype=np.int64)
        draws = g.random(100_003)
        out[f"u{i}_head"] = draws[:257]
        out[f"u{i}_tail"] = draws[-37:]
        out[f"u{i}_sum"] = np.array(draws.sum())
    keys = np.arange(10_000, dtype=np.uint64) * np.uint64(3)
    t = cpfit.SparseTensor((40_000,), keys, np.arange(10_000, dtype=np.float64))
    for j, (rate, seed, path) in enumerate([(0.01, 3, (1, 1)), (0.1, 3, (1, 2)),
                                            (0.5, 9, (1, 5)), (1.0, 1, ())]):
        s = t.sample(rate, cpfit.RngState(seed, path))
        out[f"s{j}_rate"] = np.array(rate)
        out[f"s{j}_seed"] = np.array(seed)
        out[f"s{j}_path"] = np.array(path, dtype=np.int64)
        out[f"s{j}_keys"] = s.keys
    out["n_uniform"] = np.array(len(cases))
    out["n_sample"] = np.array(4)
    np.savez_compressed(os.path.join(HERE, "philox.npz"), **out)


def cfg1():
    shape, keys, values, factors = synth.cfg1()
    t = cpfit.SparseTensor(shape, keys, values)
    out = {"keys_sha": np.array(sha(keys)), "values_sha": np.array(sha(values)),
           "factors_sha": np.array(sha(np.concatenate([f.ravel() for f in factors])))}
    out["tttp"] = rk.tttp(t, factors).values
    for mode in range(3):
        out[f"mttkrp{mode}"] = rk.mttkrp(t, factors, mode)
    loss = cpfit.get_loss("ls")
    cfg = ro.SolverConfig(rank=10, reg=1e-5)
    state = ro.CompletionState(factors=[f.copy() for f in factors], rng=cpfit.RngState(0))
    for s in range(5):
        ro.als_sweep(t, state, loss, cfg)
        for n in range(3):
            out[f"als{s}_f{n}"] = state.factors[n].copy()
        out[f"als{s}_rmse"] = np.array(cpfit.rmse(t, state.factors))
    out["als_gram2"] = state.ls_gram[2][:5].copy()
    out["als_rhs2"] = state.ls_rhs[2].copy()
    state = ro.CompletionState(factors=[f.copy() for f in factors], rng=cpfit.RngState(0))
    for s in range(2):
        ro.ccd_sweep(t, state, loss, cfg)
        for n in range(3):
            out[f"ccd{s}_f{n}"] = state.factors[n].copy()
    scfg = ro.SolverConfig(rank=10, reg=1e-4, step=1e-3, sample_rate=0.1,
                           algorithm="sgd")
    state = ro.CompletionState(factors=[f.copy() for f in factors], rng=cpfit.RngState(0))
    for it in range(1, 4):
        ro.sgd_sweep(t, state, loss, scfg, cpfit.RngState(11).child(1).child(it))
        for n in range(3):
            out[f"sgd{it}_f{n}"] = state.factors[n].copy()
    np.savez_compressed(os.path.join(HERE, "cfg1.npz"), **out)


def drivers_small():
    rng = np.random.default_rng(26)
    t = random_sparse((8, 7, 6), 0.5, rng)
    out = {"dims": np.array(t.shape), "keys": t.keys, "values": t.values}
    for algo in ("als", "ccd", "sgd"):
        cfg = ro.SolverConfig(rank=3, algorithm=algo, max_iters=4, seed=4,
                              deterministic=True, sample_rate=0.5, step=1e-3,
                              record_every=1)
        trace, state = ro.run(t, cfg, return_state=True)
        out[f"{algo}_obj"] = np.array([r.objective for r in trace.records])
        out[f"{algo}_metric"] = np.array([r.metric for r in trace.records])
        out[f"{algo}_iters"] = np.array([r.iteration for r in trace.records])
        for n in range(3):
            out[f"{algo}_f{n}"] = state.factors[n]
    np.savez_compressed(os.path.join(HERE, "drivers_small.npz"), **out)


def second_order():
    rng = np.random.default_rng(31)
    out = {}
    # implicit Hessian products on small fully observed instances
    case = 0
    for ident in ("ls", "poisson"):
        for variant in ("gauss_newton", "newton"):
            dims = (4, 3, 2) if case % 2 == 0 else (5, 3, 3, 2)
            total = int(np.prod(dims))
            keys = np.arange(total, dtype=np.uint64)
            vals = rng.random(total) * 3.0 if ident == "poisson" else \
                rng.standard_normal(total)
            t = cpfit.SparseTensor(dims, keys, vals)
            factors = [0.5 * rng.standard_normal((d, 2)) for d in dims]
            x = [rng.standard_normal((d, 2)) for d in dims]
            loss = cpfit.get_loss(ident)
            model = cpfit.model_at_observed(t.observation_mask(), factors)
            phi1, phi2 = cpfit.derivative_tensors(loss, t, model)
            reg = float(rng.random() * 0.4)
            y = ro.hessian_matvec(phi1, phi2, factors, x, variant=variant, reg=reg)
            g = ro.gradient_blocks(t, factors, loss, reg)
            out[f"hv{case}_dims"] = np.array(dims)
            out[f"hv{case}_vals"] = vals
            out[f"hv{case}_ident"] = np.array(ident)
            out[f"hv{case}_variant"] = np.array(variant)
            out[f"hv{case}_reg"] = np.array(reg)
            for n in range(len(dims)):
                out[f"hv{case}_f{n}"] = factors[n]
                out[f"hv{case}_x{n}"] = x[n]
                out[f"hv{case}_y{n}"] = y[n]
                out[f"hv{case}_g{n}"] = g[n]
            case += 1
    out["hv_cases"] = np.array(case)
    # gn_step trajectories near a low-rank truth
    t, truth = cpfit.gen_low_rank((24, 20, 16), 3, 0.4, rng=cpfit.RngState(32))
    noise = np.random.default_rng(33)
    init = [f + 0.05 * noise.standard_normal(f.shape) for f in truth]
    out["gn_dims"] = np.array(t.shape)
    out["gn_keys"] = t.keys
    out["gn_values"] = t.values
    for n in range(3):
        out[f"gn_init{n}"] = init[n]
    for tag, variant, ident, kw in (("gnls", "gauss_newton", "ls", {}),
                                    ("ntls", "newton", "ls", {}),
                                    ("gnls_damped", "gauss_newton", "ls",
                                     {"gn_damping": 0.1})):
        cfg = ro.SolverConfig(rank=3, reg=1e-4, cg_tol=1e-10, cg_max=300, **kw)
        state = ro.CompletionState(factors=[f.copy() for f in init], rng=cpfit.RngState(0))
        used = []
        for s in range(3):
            used.append(ro.gn_step(t, state, cpfit.get_loss(ident), cfg, variant=variant))
            for n in range(3):
                out[f"{tag}{s}_f{n}"] = state.factors[n].copy()
        out[f"{tag}_cg"] = np.array(used)
    # poisson: counts from the truth model
    tp = t.with_values(np.round(t.values * 4.0))
    out["gnpo_values"] = tp.values
    cfg = ro.SolverConfig(rank=3, reg=1e-3, cg_tol=1e-10, cg_max=300, loss="poisson")
    pinit = [0.3 * f for f in init]
    for n in range(3):
        out[f"gnpo_init{n}"] = pinit[n]
    state = ro.CompletionState(factors=[f.copy() for f in pinit], rng=cpfit.RngState(0))
    used = []
    for s in range(2):
        used.append(ro.gn_step(tp, state, cpfit.get_loss("poisson"), cfg))
        for n in range(3):
            out[f"gnpo{s}_f{n}"] = state.factors[n].copy()
    out["gnpo_cg"] = np.array(used)
    # run() traces
    rng2 = np.random.default_rng(26)
    ts = random_sparse((8, 7, 6), 0.5, rng2)
    for algo, kw in (("gn", {"calibrate_init": True, "gn_damping": 1.0}),
                     ("newton", {"warmup_sweeps": 1, "gn_damping": 1.0, "calibrate_init": True})):
        cfg = ro.SolverConfig(rank=3, algorithm=algo, max_iters=3, seed=4, deterministic=True,
                              record_every=1, **kw)
        trace, state = ro.run(ts, cfg, return_state=True)
        out[f"run_{algo}_obj"] = np.array([r.objective for r in trace.records])
        out[f"run_{algo}_metric"] = np.array([r.metric for r in trace.records])
        out[f"run_{algo}_iters"] = np.array([r.iteration for r in trace.records])
        for n in range(3):
            out[f"run_{algo}_f{n}"] = state.factors[n]
    np.savez_compressed(os.path.join(HERE, "second_order.npz"), **out)


def generalized():
    out = {}
    t, truth = cpfit.gen_low_rank((14, 12, 10), 3, 0.5, rng=cpfit.RngState(41))
    noise = np.random.default_rng(42)
    counts = np.round(np.exp(np.clip(t.values, -3, 3)) + noise.random(t.nnz))
    tp = t.with_values(counts)
    out["dims"] = np.array(tp.shape)
    out["keys"] = tp.keys
    out["values"] = tp.values
    init = [0.3 * f + 0.05 * noise.standard_normal(f.shape) for f in truth]
    for n in range(3):
        out[f"init{n}"] = init[n]
    # elementwise: derivative tensors and objective, with clamped entries
    loss = cpfit.get_loss("poisson")
    big = [f.copy() for f in init]
    big[0] = big[0] * 3000.0
    model = cpfit.model_at_observed(tp.observation_mask(), big)
    p1, p2 = cpfit.derivative_tensors(loss, tp, model)
    out["big0"] = big[0]
    out["clamp_phi1"] = p1.values
    out["clamp_phi2"] = p2.values
    out["clamp_count_derivs"] = np.array(loss.diagnostics["exp_clamped"])
    out["clamp_obj"] = np.array(cpfit.objective(loss, tp, big, reg=1e-3))
    out["clamp_count_total"] = np.array(loss.diagnostics["exp_clamped"])
    # sweeps
    for algo, nsweep, kw in (("als", 2, {}), ("als_frozen", 2, {"freeze_curvature": True}),
                             ("ccd", 2, {}), ("sgd", 3, {"sample_rate": 0.5, "step": 1e-2})):
        loss = cpfit.get_loss("poisson")
        cfg = ro.SolverConfig(rank=3, reg=1e-3, loss="poisson", **kw)
        state = ro.CompletionState(factors=[f.copy() for f in init], rng=cpfit.RngState(0))
        for s in range(nsweep):
            if algo.startswith("als"):
                ro.als_sweep(tp, state, loss, cfg)
            elif algo == "ccd":
                ro.ccd_sweep(tp, state, loss, cfg)
            else:
                ro.sgd_sweep(tp, state, loss, cfg, cpfit.RngState(5).child(s))
            for n in range(3):
                out[f"{algo}{s}_f{n}"] = state.factors[n].copy()
    # least squares through the generalized (inner Newton) ALS path
    loss = cpfit.get_loss("ls")
    cfg = ro.SolverConfig(rank=3, reg=1e-3)
    state = ro.CompletionState(factors=[f.copy() for f in init], rng=cpfit.RngState(0))
    ro.als_sweep(t, state, loss, cfg, generalized=True)
    out["lsgen_values"] = t.values
    for n in range(3):
        out[f"lsgen_f{n}"] = state.factors[n].copy()
    # run() traces
    for algo in ("als", "ccd", "sgd"):
        cfg = ro.SolverConfig(rank=3, algorithm=algo, loss="poisson", max_iters=3, seed=4,
                              deterministic=True, record_every=1, sample_rate=0.5, step=1e-2)
        trace, state = ro.run(tp, cfg, return_state=True)
        out[f"run_{algo}_obj"] = np.array([r.objective for r in trace.records])
        out[f"run_{algo}_metric"] = np.array([r.metric for r in trace.records])
        for n in range(3):
            out[f"run_{algo}_f{n}"] = state.factors[n]
    np.savez_compressed(os.path.join(HERE, "generalized.npz"), **out)


def ingest():
    from cpfit import tensor_io as rio
    rng = np.random.default_rng(51)
    out = {}
    shape = (50, 40, 30)
    n = 80_000
    c = [rng.integers(0, d, n).astype(np.int32) for d in shape]
    for q, v in enumerate((7, 11, 13)):
        c[q][:3000] = v          # one key 3000 times (recursive pairwise halves)
    for q, v in enumerate((1, 2, 3)):
        c[q][3000:3100] = v      # one key 100 times (eight accumulators)
    vals = rng.standard_normal(n) * 10.0 ** rng.integers(-6, 7, n)
    perm = rng.permutation(n)
    c = [x[perm] for x in c]
    vals = vals[perm]
    t = cpfit.from_coords(c, vals, shape)
    out["a_shape"] = np.array(shape)
    for q in range(3):
        out[f"a_c{q}"] = c[q]
    out["a_vals"] = vals
    out["a_keys"] = t.keys
    out["a_out"] = t.values
    shape4 = (100_000, 100_000, 100_000, 1000)
    m = 40_000
    c4 = [rng.integers(0, d, m).astype(np.int32) for d in shape4]
    v4 = rng.standard_normal(m)
    t4 = cpfit.from_coords(c4, v4, shape4)
    out["b_shape"] = np.array(shape4)
    for q in range(4):
        out[f"b_c{q}"] = c4[q]
    out["b_vals"] = v4
    out["b_keys"] = t4.keys
    out["b_out"] = t4.values
    lines = ["# a comment", "# dims: 9 8 7"]
    for _ in range(400):
        i, j, k = (int(rng.integers(1, 10)), int(rng.integers(1, 9)), int(rng.integers(1, 8)))
        lines.append(f"{i} {j} {k} {rng.standard_normal()!r}")
    text = "\n".join(lines) + "\n"
    path = "/tmp/cpfit_golden.tns"
    with open(path, "w") as fh:
        fh.write(text)
    tt = rio.parse_tns(path)
    out["tns_text"] = np.array(text)
    out["tns_shape"] = np.array(tt.shape)
    out["tns_keys"] = tt.keys
    out["tns_vals"] = tt.values
    np.savez_compressed(os.path.join(HERE, "ingest.npz"), **out)


def _ccsr_out(out, tag, a):
    out[f"{tag}_shape"] = np.array([a.global_rows, a.global_cols])
    out[f"{tag}_rows"] = a.nnz_row_ids
    out[f"{tag}_offs"] = a.row_offsets
    out[f"{tag}_cols"] = a.col_ids
    out[f"{tag}_vals"] = a.values


def hypersparse():
    from cpfit import hypersparse as H
    rng = np.random.default_rng(61)
    out = {}
    # COO -> CCSR (distinct pairs, shuffled)
    gr, gc = 100_000, 300
    keys = np.unique(rng.integers(0, gr * gc, 5000))
    rng.shuffle(keys)
    r, c = keys // gc, keys % gc
    v = rng.standard_normal(keys.size)
    a = H.ccsr_from_coo(r, c, v, gr, gc)
    out["coo_r"], out["coo_c"], out["coo_v"] = r, c, v
    _ccsr_out(out, "coo", a)
    # matricize: native and permuted
    t = random_sparse((9, 8, 7, 6), 0.2, rng)
    out["t_dims"], out["t_keys"], out["t_vals"] = np.array(t.shape), t.keys, t.values
    for tag, rm, cm in (("mat_native", (0, 1), (2, 3)), ("mat_perm", (3, 1), (0, 2)),
                        ("mat_rowsonly", (2, 0, 3, 1), ())):
        _ccsr_out(out, tag, H.matricize_to_ccsr(t, rm, cm))
    # CCSR x dense
    b = rng.standard_normal((gc, 7))
    out["spmm_b"] = b
    z = H.ccsr_times_dense(a, b)
    out["spmm_keys"], out["spmm_payload"] = z.fiber_keys, z.payload
    # sums with cancellations
    a2 = H.ccsr_from_coo(r[:2000], c[:2000], -v[:2000], gr, gc)
    keys3 = np.unique(rng.integers(0, gr * gc, 3000))
    a3 = H.ccsr_from_coo(keys3 // gc, keys3 % gc, rng.standard_normal(keys3.size), gr, gc)
    _ccsr_out(out, "a2", a2)
    _ccsr_out(out, "a3", a3)
    _ccsr_out(out, "sum12", H.ccsr_sum(a, a2))
    _ccsr_out(out, "sum13", H.ccsr_sum(a, a3))
    # butterfly reduce-scatter of 5 summands
    parts = []
    for p_ in range(5):
        kk = np.unique(rng.integers(0, 40 * 50, 300))
        parts.append(H.ccsr_from_coo(kk // 50, kk % 50, rng.standard_normal(kk.size), 40, 50))
        _ccsr_out(out, f"bf_in{p_}", parts[-1])
    for k in (2, 3):
        for canon in (True, False):
            shards = H.butterfly_reduce_scatter(parts, k=k, canonical=canon)
            for p_, sh in enumerate(shards):
                _ccsr_out(out, f"bf_k{k}_c{int(canon)}_s{p_}", sh)
            _ccsr_out(out, f"bf_k{k}_c{int(canon)}_all", H.butterfly_gather(shards))
    # ttm / pairwise
    w = rng.standard_normal((t.shape[2], 5))
    out["ttm_w"] = w
    zz = H.ttm(t, w, 2)
    out["ttm_keys"], out["ttm_payload"] = zz.fiber_keys, zz.payload
    f4 = [rng.standard_normal((d, 5)) for d in t.shape]
    for n in range(4):
        out[f"pw_f{n}"] = f4[n]
    for mode in range(4):
        out[f"pw_mttkrp{mode}"] = H.pairwise_mttkrp(t, f4, mode)
    t3 = random_sparse((11, 10, 9), 0.3, rng)
    out["t3_dims"], out["t3_keys"], out["t3_vals"] = np.array(t3.shape), t3.keys, t3.values
    for R in (1, 7, 8, 20):
        fs = [rng.standard_normal((d, R)) for d in t3.shape]
        for n in range(3):
            out[f"pt{R}_f{n}"] = fs[n]
        out[f"pt{R}_out"] = H.pairwise_tttp(t3, fs).values
        out[f"pt{R}_none_out"] = H.pairwise_tttp(t3, [None, fs[1], fs[2]]).values
        out[f"pt{R}_mttkrp1"] = H.pairwise_mttkrp(t3, fs, 1)
    np.savez_compressed(os.path.join(HERE, "hypersparse.npz"), **out)


def cli():
    import subprocess
    import tempfile
    env = dict(os.environ, PYTHONPATH="/root/reference/pkg/src")
    out = {}
    with tempfile.TemporaryDirectory() as d:
        data = os.path.join(d, "x.tns")
        subprocess.run([sys.executable, "-m", "cpfit", "gen", "lowrank", "--dims", "12,12,12",
                        "--rank", "3", "--fraction", "0.3", "--seed", "5", "--out", data],
                       check=True, env=env, capture_output=True)
        out["gen_tns"] = np.array(open(data).read())
        out["gen_factors"] = np.frombuffer(open(data + ".factors.npy", "rb").read(), np.uint8)
        pdata = os.path.join(d, "p.tns")
        subprocess.run([sys.executable, "-m", "cpfit", "gen", "function", "--dims", "8,7,6",
                        "--fraction", "0.5", "--seed", "2", "--out", pdata],
                       check=True, env=env, capture_output=True)
        out["gen_function_tns"] = np.array(open(pdata).read())
        runs = {"als": ["--algo", "als"], "ccd": ["--algo", "ccd"],
                "sgd": ["--algo", "sgd", "--sample-rate", "0.5", "--step", "0.01"],
                "gn": ["--algo", "gn"],
                "als_poisson": ["--algo", "als", "--loss", "poisson"]}
        for tag, extra in runs.items():
            tr = os.path.join(d, f"{tag}.csv")
            src = pdata if tag.endswith("poisson") else data
            subprocess.run([sys.executable, "-m", "cpfit", "run", "--input", src, "--rank", "3",
                            "--max-iters", "5", "--seed", "11", "--deterministic",
                            "--trace", tr, *extra], check=True, env=env, capture_output=True)
            out[f"trace_{tag}"] = np.array(open(tr).read())
    np.savez_compressed(os.path.join(HERE, "cli.npz"), **out)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        for name in sys.argv[1:]:
            globals()[name]()
        sys.exit(0)
    kernels_small()
    layout()
    philox()
    cfg1()
    drivers_small()
    generalized()
    ingest()
    hypersparse()
    cli()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
