"""The pybind-surface front-end (paper_2603_16014_b200/fastmtgp.py, bindings.cpp:129-213) and the
model document I/O (gp_core.cpp:447-508).  CPU tests: design ordering / shift streams, weights,
document checks; GPU tests: the Model against the reference library on the same design."""
import json

import numpy as np
import pytest

from paper_2603_16014_b200 import fastmtgp
from paper_2603_16014_b200._lib import Unsupported
from paper_2603_16014_b200.designs import DIGITAL, LATTICE


def test_make_design_user_order_and_streams():
    """Internal order = stable descending size (ld_sequences.cpp:175-176); the shift of a task
    follows its USER index, so reordering the other tasks does not change it."""
    d1, i2u1 = fastmtgp.make_design(LATTICE, 3, [5, 7, 5, 6], seed=9)
    assert i2u1 == [1, 3, 0, 2] and d1.m == [7, 6, 5, 5]
    d2, i2u2 = fastmtgp.make_design(LATTICE, 3, [5, 7], seed=9)
    assert i2u2 == [1, 0]
    assert np.array_equal(d1.shift_bits[0], d2.shift_bits[0])  # both: user task 1
    assert not np.array_equal(d1.shift_bits[0], d1.shift_bits[2])
    pts = fastmtgp.design_points("digital", 2, [8, 32, 16], seed=4)
    assert [p.shape for p in pts] == [(8, 2), (32, 2), (16, 2)]
    assert all(np.all((p >= 0) & (p < 1)) for p in pts)


def test_optimal_weights_formula():
    rng = np.random.default_rng(1)
    A = rng.standard_normal((3, 3))
    Sigma, mu, chi = A @ A.T + np.eye(3), rng.standard_normal(3), np.array([1.0, 0.0, 0.0])
    w, mse = fastmtgp.optimal_weights(mu, Sigma, chi)
    # the minimiser of w^T Sigma w + (w.mu - chi.mu)^2 (cubature.cpp weights_mse)
    f = lambda v: v @ Sigma @ v + (v @ mu - chi @ mu) ** 2  # noqa: E731
    assert abs(f(w) - mse) <= 1e-12 * max(1.0, abs(mse))
    for _ in range(5):
        assert f(w + 1e-3 * rng.standard_normal(3)) >= f(w)


def test_reference_document_without_generator_is_rejected():
    doc = {"kind": "lattice", "family": "si-lattice", "loss": "nmll", "d": 2, "seed": 1, "m": [3],
           "hyper": {"gamma": 1.0, "eta": [1, 1], "si_alpha": 1, "b": [1, 1, 1, 1], "t": [0.1], "xi": [1e-8],
                     "tau": [0.0], "lengthscales": [0.25, 0.25], "B": [[0.1]]}, "y": [[0.0] * 8]}
    with pytest.raises(Unsupported):
        fastmtgp.Model.from_json(json.dumps(doc))


def test_se_dense_is_unsupported():
    with pytest.raises(Unsupported):
        fastmtgp.Model("se-dense", 2, [8], 1, [[0.0] * 8])


@pytest.mark.gpu
@pytest.mark.parametrize("kernel,n", [("si-lattice", [64, 256]), ("dsi-digital", [32, 128, 32])])
def test_model_matches_reference(ref, kernel, n):
    rng = np.random.default_rng(5)
    y = [rng.standard_normal(v) for v in n]
    m = fastmtgp.Model(kernel, 3, n, seed=11, y=y, task_rank=1, jitter=1e-6)
    hi = m._internal(m.hyper)
    yi = np.concatenate([y[u] for u in m.i2u])
    rm = ref.Model(m.design, hi, yi)
    want = rm.loss(0)
    assert abs(m.loss() - want) <= 1e-8 * m.design.N
    st = rm.state()
    assert np.allclose(m.tau(), m._uvec(st["tau"]), rtol=1e-10, atol=1e-12)
    X = np.random.default_rng(2).random((5, 3))
    for u in range(len(n)):
        got = m.posterior_mean_batch(u, X)
        exp = rm.posterior_mean(m.i2u.index(u), X)
        assert np.allclose(got, exp, rtol=1e-9, atol=1e-12)
    c = m.posterior_cov(0, X[0], len(n) - 1, X[1])
    c_ref = rm.posterior_cov(m.i2u.index(0), X[0], m.i2u.index(len(n) - 1), X[1])
    assert abs(c - c_ref) <= 1e-8 * max(1.0, abs(c_ref))
    mu, S = m.cubature()
    mur, Sr = rm.cubature()
    assert np.allclose(mu, m._uvec(mur), rtol=1e-9, atol=1e-12)
    assert np.allclose(S, m._umat(Sr), rtol=1e-8, atol=1e-12)


@pytest.mark.gpu
def test_fit_and_json_round_trip():
    rng = np.random.default_rng(8)
    n = [128, 64]
    m = fastmtgp.Model("si-lattice", 2, n, seed=3, y=[rng.standard_normal(v) for v in n])
    rep = m.fit(5)
    assert len(rep["loss_trace"]) == 5 and np.all(np.diff(rep["loss_trace"]) <= 0)
    doc = m.to_json()
    m2 = fastmtgp.Model.from_json(doc)
    assert m2.loss() == pytest.approx(m.loss(), rel=1e-13)
    assert json.loads(m2.to_json()) == json.loads(doc)


def test_cli_points(tmp_path):
    from paper_2603_16014_b200 import cli
    out = tmp_path / "pts.csv"
    assert cli.main(["points", "--kernel", "si-lattice", "--n", "16,4", "--d", "3", "--seed", "5", "--out", str(out)]) == 0
    rows = out.read_text().strip().splitlines()
    assert rows[0] == "task,index,x1,x2,x3" and len(rows) == 1 + 16 + 4
    pts = fastmtgp.design_points("lattice", 3, [16, 4], 5)
    first = [float(v) for v in rows[1].split(",")[2:]]
    assert first == list(pts[0][0])


@pytest.mark.gpu
def test_cli_fit_and_cubature(tmp_path):
    from paper_2603_16014_b200 import cli
    rng = np.random.default_rng(4)
    n = [64, 32]
    m = fastmtgp.Model("dsi-digital", 2, n, seed=9, y=[rng.standard_normal(v) for v in n])
    doc = tmp_path / "m.json"
    doc.write_text(m.to_json())
    rep, cub, fitted = tmp_path / "rep.json", tmp_path / "cub.json", tmp_path / "fitted.json"
    assert cli.main(["fit", "--model", str(doc), "--steps", "3", "--model-out", str(fitted), "--out", str(rep)]) == 0
    r = json.loads(rep.read_text())
    assert len(r["loss_trace"]) == 3 and r["loss"] <= r["loss_trace"][0] + 1e-9 * abs(r["loss_trace"][0])
    assert cli.main(["cubature", "--model", str(fitted), "--out", str(cub)]) == 0
    c = json.loads(cub.read_text())
    assert len(c["mu"]) == 2 and len(c["Sigma"]) == 2


def test_test_points_and_problem_errors():
    """The held-out set (bench.cpp:155-157): generator points under the test-stream shift — in the
    unit cube, distinct from the design's own points; problem arguments checked before the device."""
    X = fastmtgp.test_points("si-lattice", 4, 256, seed=3)
    assert X.shape == (256, 4) and np.all((X >= 0) & (X < 1))
    D = fastmtgp.design_points("lattice", 4, [256], 3)[0]
    assert not np.allclose(X, D)
    Xd = fastmtgp.test_points("dsi-digital", 2, 64, seed=3)
    assert Xd.shape == (64, 2) and len(np.unique(Xd[:, 0])) == 64
    with pytest.raises(ValueError):
        fastmtgp.Model.from_problem("nosuch", "si-lattice", [64])
    with pytest.raises(ValueError):
        fastmtgp.Model.from_problem("ackley", "si-lattice", [64, 32, 16])  # ackley has 2 fidelities
    with pytest.raises(Unsupported):
        fastmtgp.Model.from_problem("ackley", "se-dense", [64])


@pytest.mark.gpu
@pytest.mark.parametrize("kernel", ["si-lattice", "dsi-digital"])
def test_model_from_problem(ref, kernel):
    """fit_trial on a benchmark problem (bench.cpp:84-107): device observations equal the
    reference's functions at the design points plus the noise stream; fitting lowers the loss and
    the held-out l2 error of the top fidelity is small on a smooth problem."""
    n = [1024, 256]
    m = fastmtgp.Model.from_problem("ackley", kernel, n, seed=2, noise=1e-4)
    for u in range(2):
        want = ref.problem_eval("ackley", u + 1, fastmtgp.design_points(
            "lattice" if kernel == "si-lattice" else "digital", 4, n, 2)[u])
        assert np.abs(m.y_user[u] - want).max() <= 1e-3  # noise 1e-4 * N(0,1)
    l0 = m.loss()
    rep = m.fit(8)
    assert m.loss() <= l0 and len(rep["loss_trace"]) == 8
    X = fastmtgp.test_points(kernel, 4, 512, seed=2)
    errs = [m.l2_relative_error(u, X) for u in range(2)]
    assert all(np.isfinite(errs)) and errs[0] < 0.5, errs


@pytest.mark.gpu
def test_cli_problem_fit_cubature_bench(tmp_path):
    from paper_2603_16014_b200 import cli
    rep, cub, bench = tmp_path / "r.json", tmp_path / "c.json", tmp_path / "b.csv"
    assert cli.main(["fit", "--problem", "rosenbrock", "--kernel", "si-lattice", "--n", "256,64,16", "--steps", "4",
                     "--noise", "1e-3", "--test-points", "128", "--out", str(rep)]) == 0
    r = json.loads(rep.read_text())
    assert r["n"] == "256x64x16" and len(r["l2_rel_error"]) == 3 and len(r["report"]["loss_trace"]) == 4
    assert cli.main(["cubature", "--problem", "borehole", "--n", "128,32", "--steps", "3", "--out", str(cub)]) == 0
    c = json.loads(cub.read_text())
    assert len(c["mu"]) == 2 and len(c["weights"]) == 2 and c["problem"] == "borehole"
    assert cli.main(["bench", "--problem", "ackley", "--n", "128,64", "--steps", "3", "--trials", "2",
                     "--test-points", "64", "--out", str(bench)]) == 0
    rows = bench.read_text().strip().splitlines()
    assert rows[0].startswith("problem,method,n,trial") and len(rows) == 4 and rows[-1].split(",")[3] == "median"
