"""GPU parity of the `run_experiment` drop-in (reference harness.py:188-289)
against the reference's own ExperimentReport rows (tests/golden/experiment.npz,
made by tests/golden/make_golden_experiment.py), and of the drop-in payload
policy: numpy in -> numpy out, consumed unchanged by the reference-restated
`match_eigenvectors` (sequence.py:187-220) and by `emit_report`."""

import json
import os

import numpy as np
import pytest
import torch

import paper_1206_3768_b200 as pkg
from oracle import chfsi_oracle as orc
from paper_1206_3768_b200 import sequence
from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def exp_golden():
    return np.load(os.path.join(GOLDEN, "experiment.npz"))


def _specs(g):
    for name in g["names"]:
        name = str(name)
        yield name, json.loads(bytes(g[f"{name}/spec"]))


def _spec(sp, reps=1):
    sched = pkg.CorrelationSchedule(**sp["schedule"])
    return pkg.ExperimentSpec(source=pkg.GenerateSource(n=sp["n"], schedule=sched, seed=sp["seed"]),
                              solver="chfsi", nev=sp["nev"], solver_overrides=sp["overrides"],
                              tracked_fraction=sp["fraction"], repetitions=reps, seed=sp["seed"])


def test_run_experiment_matches_reference_rows(exp_golden, tmp_path):
    for name, sp in _specs(exp_golden):
        rep = pkg.run_experiment(_spec(sp))
        g = {k[len(name) + 1:]: exp_golden[k] for k in exp_golden.files if k.startswith(name + "/")}
        assert rep.blk == int(g["blk"]) and rep.length == sp["schedule"]["length"]
        assert rep.warnings == json.loads(bytes(g["warnings"]))
        assert [r.ell for r in rep.rows] == g["ell"].tolist()
        tol = sp["overrides"].get("tol", 1e-10)
        deg = sp["overrides"].get("deg", 25)
        for i, r in enumerate(rep.rows):
            for kind in ("random", "approx"):
                loops = getattr(r, f"inner_loops_{kind}")
                assert abs(loops - int(g[f"inner_loops_{kind}"][i])) <= 1, (name, r)
                if loops == int(g[f"inner_loops_{kind}"][i]):  # same passes: same counts
                    assert getattr(r, f"matvecs_{kind}") == int(g[f"matvecs_{kind}"][i])
                    assert getattr(r, f"filtered_{kind}") == int(g[f"filtered_{kind}"][i])
                else:
                    assert abs(getattr(r, f"matvecs_{kind}") - int(g[f"matvecs_{kind}"][i])) \
                        <= (deg + 1) * rep.blk
                assert getattr(r, f"converged_{kind}") == bool(g[f"converged_{kind}"][i])
                assert getattr(r, f"max_residual_{kind}") <= tol
            # dense eigenvectors of adjacent problems: same matching medians
            assert r.median_angle == pytest.approx(float(g["median_angle"][i]), rel=1e-6, abs=1e-12)
        pkg.emit_report(rep, "csv", tmp_path / f"{name}.csv")
        header = (tmp_path / f"{name}.csv").read_text().splitlines()[0].split(",")
        assert header == [str(x) for x in exp_golden["report_fields"]]


def test_run_experiment_repetitions_and_sources(tmp_path):
    """repetitions > 1 re-solves with the same seeds (identical counts), the
    BASELINE and saved-directory sources run the same protocol, and a
    1-problem sequence only warns (harness.py:205-208)."""
    src = pkg.BaselineSource(n=160, length=3, seed=0)
    spec = pkg.ExperimentSpec(source=src, solver="chfsi", nev=8,
                              solver_overrides=dict(nex=8, deg=10), repetitions=2)
    rep = pkg.run_experiment(spec)
    assert rep.all_converged and len(rep.rows) == 2
    assert all(r.speedup_matvec > 1.0 for r in rep.rows)
    pkg.save_sequence(pkg.iter_baseline_sequence(160, 3, seed=0), tmp_path / "seq")
    rep2 = pkg.run_experiment(pkg.ExperimentSpec(source=pkg.LoadSource(str(tmp_path / "seq")),
                                                 solver="chfsi", nev=8,
                                                 solver_overrides=dict(nex=8, deg=10),
                                                 repetitions=1))
    assert [(r.matvecs_random, r.matvecs_approx) for r in rep2.rows] == \
        [(r.matvecs_random, r.matvecs_approx) for r in rep.rows]
    one = pkg.run_experiment(pkg.ExperimentSpec(source=pkg.BaselineSource(n=64, length=1),
                                                solver="chfsi", nev=4, repetitions=1))
    assert one.rows == [] and one.warnings
    with pytest.raises(ValueError, match="blk < n"):
        pkg.run_experiment(pkg.ExperimentSpec(source=pkg.BaselineSource(n=40, length=2),
                                              solver="chfsi", nev=4, repetitions=1))


@pytest.mark.host_payloads
def test_numpy_payloads_feed_reference_consumers(exp_golden):
    """Drop-in default: numpy inputs give numpy outputs, and the reference's
    consumers (the restated match_eigenvectors argmax loop, numpy
    arithmetic on the vectors) run on them unchanged."""
    name, sp = next(_specs(exp_golden))
    sched = pkg.CorrelationSchedule(**sp["schedule"])
    blk = int(exp_golden[f"{name}/blk"])
    keep = max(blk + 1, sp["nev"])
    tracked = max(1, int(np.ceil(sp["fraction"] * sp["nev"])))
    sols = []
    for lab, a, b in sequence.iter_generated_sequence(sp["n"], sched, sp["seed"]):
        pencil = pkg.EigenPencil(a=a, b=b, label=lab)
        sol, stdp, vals = pkg.oracle_solve(pencil, keep)
        assert isinstance(sol.vectors, np.ndarray) and isinstance(stdp.h, np.ndarray)
        assert isinstance(stdp.cholesky_factor, np.ndarray)
        sols.append(sol)
        # ChFSI on the numpy operator: numpy vectors, numpy residual arithmetic
        csol, crep = pkg.chfsi_solve(stdp.h, pkg.ChfsiConfig(nev=sp["nev"], **sp["overrides"]),
                                     rng=np.random.default_rng((sp["seed"], lab, 0)))
        assert isinstance(csol.vectors, np.ndarray) and crep.converged
        r = stdp.h @ csol.vectors - csol.vectors * csol.values
        assert np.linalg.norm(r, axis=0).max() <= 1e-9
        gsol = pkg.back_transform(stdp.cholesky_factor, csol)
        assert isinstance(gsol.vectors, np.ndarray)
        assert np.abs(a @ gsol.vectors - (b @ gsol.vectors) * csol.values).max() <= 1e-8
        y = np.random.default_rng(1).standard_normal((sp["n"], 5)) + 0j
        f = pkg.chebyshev_filter(stdp.h, y, 4, pkg.FilterWindow(a=float(vals[blk]),
                                                                b=float(vals[-1]) + 0.1,
                                                                scale_ref=float(vals[0])))
        assert isinstance(f, np.ndarray)
        ref = orc.chebyshev_filter(stdp.h, y, 4, float(vals[blk]), float(vals[-1]) + 0.1,
                                   float(vals[0]))
        assert np.abs(f - ref).max() <= 1e-12 * np.abs(ref).max()
    for i in range(len(sols) - 1):
        ya, yb = sols[i].vectors[:, :tracked], sols[i + 1].vectors[:, :tracked]
        sigma, theta = orc.match_eigenvectors(ya, yb)
        np.testing.assert_array_equal(sigma, exp_golden[f"{name}/sigma/{i + 1}"])
        np.testing.assert_allclose(theta, exp_golden[f"{name}/theta/{i + 1}"], rtol=1e-6, atol=1e-9)
        s2, t2 = pkg.match_eigenvectors(pkg.EigenSolution(sols[i].values[:tracked], ya),
                                        None, pkg.EigenSolution(sols[i + 1].values[:tracked], yb),
                                        None)
        np.testing.assert_array_equal(s2, sigma)
        np.testing.assert_allclose(t2, theta, rtol=1e-9, atol=1e-12)
    # CUDA-tensor inputs keep the outputs in HBM under the same default policy
    hd = torch.from_numpy(np.asarray(sols[0].vectors[:, :3])).cuda()
    q = pkg.qr_orthonormalize(hd)
    assert isinstance(q, torch.Tensor) and q.is_cuda
    assert isinstance(pkg.qr_orthonormalize(sols[0].vectors[:, :3]), np.ndarray)
