"""Command-line driver (cli.py): `gen` output byte-identical to the
reference's (CPU), usage / data-error exit codes (CPU); `run` traces against
the reference's own traces, byte-stable across repeats, and `bench` (GPU)."""

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, golden

from paper_1910_02371_b200.tensor_io import read_trace


def cli(args, cwd=None):
    env = dict(os.environ, PYTHONPATH=ROOT)
    return subprocess.run([sys.executable, "-m", "paper_1910_02371_b200", *args],
                          capture_output=True, text=True, env=env, cwd=cwd)


def test_gen_bytes_match_reference(tmp_path):
    z = golden("cli")
    out = tmp_path / "x.tns"
    r = cli(["gen", "lowrank", "--dims", "12,12,12", "--rank", "3", "--fraction", "0.3",
             "--seed", "5", "--out", str(out)])
    assert r.returncode == 0, r.stderr
    assert out.read_text() == str(z["gen_tns"])
    assert np.array_equal(np.frombuffer((tmp_path / "x.tns.factors.npy").read_bytes(), np.uint8),
                          z["gen_factors"])
    out2 = tmp_path / "p.tns"
    r = cli(["gen", "function", "--dims", "8,7,6", "--fraction", "0.5", "--seed", "2",
             "--out", str(out2)])
    assert r.returncode == 0, r.stderr
    assert out2.read_text() == str(z["gen_function_tns"])


def test_usage_and_data_errors(tmp_path):
    assert cli([]).returncode == 1
    assert cli(["gen", "lowrank", "--dims", "0,3", "--out", "x"]).returncode == 1
    data = tmp_path / "x.tns"
    data.write_text("1 1 1 1.0\n")
    r = cli(["run", "--input", str(data), "--step", "0.1"])
    assert r.returncode == 1 and "--step requires --algo sgd" in r.stderr
    r = cli(["run", "--input", str(data), "--cg-tol", "0.1"])
    assert r.returncode == 1 and "requires --algo gn or newton" in r.stderr
    bad = tmp_path / "bad.tns"
    bad.write_text("1 1 1 1.0\n1 x 1 2.0\n")
    r = cli(["run", "--input", str(bad)])
    assert r.returncode == 2 and "data error" in r.stderr and ":2" in r.stderr


def _trace_values(text, path):
    path.write_text(text)
    tr = read_trace(path)
    return (tr.metric_name, tr.metadata,
            np.array([(r.iteration, r.objective, r.metric) for r in tr.records]))


@pytest.mark.gpu
@pytest.mark.parametrize("tag,extra", [
    ("als", ["--algo", "als"]), ("ccd", ["--algo", "ccd"]),
    ("sgd", ["--algo", "sgd", "--sample-rate", "0.5", "--step", "0.01"]),
    ("gn", ["--algo", "gn"]), ("als_poisson", ["--algo", "als", "--loss", "poisson"])])
def test_run_traces_match_reference_and_are_byte_stable(tmp_path, tag, extra):
    z = golden("cli")
    data = tmp_path / "d.tns"
    data.write_text(str(z["gen_function_tns"] if tag.endswith("poisson") else z["gen_tns"]))
    outs = []
    for i in range(2):
        tr = tmp_path / f"t{i}.csv"
        r = cli(["run", "--input", str(data), "--rank", "3", "--max-iters", "5", "--seed", "11",
                 "--deterministic", "--trace", str(tr), *extra])
        assert r.returncode == 0, r.stderr
        outs.append(tr.read_bytes())
    assert outs[0] == outs[1]
    name, meta, vals = _trace_values(outs[0].decode(), tmp_path / "a.csv")
    rname, rmeta, rvals = _trace_values(str(z[f"trace_{tag}"]), tmp_path / "b.csv")
    assert name == rname and meta == rmeta
    assert vals.shape == rvals.shape
    assert np.array_equal(vals[:, 0], rvals[:, 0])
    tol = 1e-8 if tag == "gn" else 1e-10
    assert np.allclose(vals[:, 1:], rvals[:, 1:], rtol=tol, atol=0)


@pytest.mark.gpu
def test_bench_smoke():
    for kernel in ("mttkrp", "tttp", "solvefactor"):
        r = cli(["bench", kernel, "--dims", "12,12,12", "--nnz", "400", "--rank", "4",
                 "--repeats", "2"])
        assert r.returncode == 0, r.stderr
        if kernel != "solvefactor":
            assert "all-at-once" in r.stdout and "pairwise" in r.stdout and "ratio" in r.stdout
