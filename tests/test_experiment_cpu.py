"""CPU tests of the run_experiment drop-in's host side: the reference
generator restatement (bytes vs the reference's, tests/golden/experiment.npz),
ExperimentSpec validation, emit_report's schema, the oracle's matcher vs the
reference's, and the array-payload policy (reference harness.py:88-336,
sequence.py:36-220)."""

import csv
import json
import os

import numpy as np
import pytest
import torch

import paper_1206_3768_b200 as pkg
from oracle import chfsi_oracle as orc
from paper_1206_3768_b200 import _device, harness, sequence
from tests.conftest import GOLDEN
from tests.golden.recipes import sha


@pytest.fixture(scope="module")
def exp_golden():
    return np.load(os.path.join(GOLDEN, "experiment.npz"))


def _specs(g):
    for name in g["names"]:
        name = str(name)
        yield name, json.loads(bytes(g[f"{name}/spec"]))


def _host_hpd(b):  # the device potrf probe, restated with numpy for the CPU suite
    try:
        np.linalg.cholesky(b)
    except np.linalg.LinAlgError:
        return False
    return True


def test_generator_reproduces_reference_bytes(exp_golden, monkeypatch):
    monkeypatch.setattr(sequence, "_b_is_hpd", _host_hpd)
    for name, sp in _specs(exp_golden):
        sched = pkg.CorrelationSchedule(**sp["schedule"])
        labels = []
        for lab, a, b in sequence.iter_generated_sequence(sp["n"], sched, sp["seed"]):
            labels.append(lab)
            np.testing.assert_array_equal(a[::7, ::5], exp_golden[f"{name}/a_probe/{lab}"])
            np.testing.assert_array_equal(b[::7, ::5], exp_golden[f"{name}/b_probe/{lab}"])
            assert sha(a) == str(bytes(exp_golden[f"{name}/a_sha/{lab}"]), "ascii")
            assert sha(b) == str(bytes(exp_golden[f"{name}/b_sha/{lab}"]), "ascii")
        assert labels == list(range(1, sched.length + 1))


def test_schedule_validation():
    s = pkg.CorrelationSchedule(length=4)
    assert s.eps == [0.5, 0.5 * 0.45, 0.5 * 0.45 ** 2]
    assert pkg.CorrelationSchedule.geometric(3, eps0=0.2, decay=0.5).eps == [0.2, 0.1]
    for bad in (dict(length=0), dict(length=3, eps=[0.1]), dict(length=2, eps=[-1.0]),
                dict(length=2, b_cond_target=0.5)):
        with pytest.raises(ValueError):
            pkg.CorrelationSchedule(**bad)
    with pytest.raises(ValueError):
        pkg.CorrelationSchedule.geometric(3, decay=1.5)
    with pytest.raises(ValueError):
        next(sequence.iter_generated_sequence(3, s))


def test_experiment_spec_validation():
    src = pkg.GenerateSource(n=32, schedule=pkg.CorrelationSchedule(length=2))
    assert pkg.SOLVERS == ("chfsi", "lobpcg", "lobpcg-generalized")
    for bad in (dict(solver="davidson"), dict(repetitions=0), dict(tracked_fraction=0.0),
                dict(tracked_fraction=1.5), dict(nev=0)):
        kw = dict(source=src, solver="chfsi", nev=4)
        kw.update(bad)
        with pytest.raises(ValueError):
            pkg.ExperimentSpec(**kw)
    spec = pkg.ExperimentSpec(source=src, solver="lobpcg", nev=4)
    with pytest.raises(NotImplementedError, match="ChFSI path only"):
        pkg.run_experiment(spec)


def _fake_report():
    rows = [harness.ExperimentRow(ell=l, t_random_s=0.5, t_approx_s=0.25, speedup_time=2.0,
                                  matvecs_random=300, matvecs_approx=200, speedup_matvec=1.5,
                                  filtered_random=40, filtered_approx=20, inner_loops_random=4,
                                  inner_loops_approx=2, median_angle=1e-3,
                                  max_residual_random=1e-11, max_residual_approx=2e-11,
                                  converged_random=True, converged_approx=l != 3)
            for l in (2, 3)]
    return harness.ExperimentReport(rows=rows, n=64, length=3, solver="chfsi", nev=4, blk=8,
                                    repetitions=1, tracked_fraction=1.0, seed=0)


def test_emit_report_schema(exp_golden, tmp_path):
    ref_fields = [str(x) for x in exp_golden["report_fields"]]
    assert pkg.REPORT_FIELDS == ref_fields
    rep = _fake_report()
    assert not rep.all_converged
    pkg.emit_report(rep, "csv", tmp_path / "r.csv")
    with open(tmp_path / "r.csv") as fh:
        rows = list(csv.DictReader(fh))
    assert list(rows[0].keys()) == ref_fields and [r["ell"] for r in rows] == ["2", "3"]
    pkg.emit_report(rep, "json", tmp_path / "r.json")
    recs = json.load(open(tmp_path / "r.json"))
    assert [list(r) for r in recs] == [ref_fields] * 2 and recs[1]["matvecs_approx"] == 200
    with pytest.raises(ValueError):
        pkg.emit_report(rep, "xml", tmp_path / "r.xml")


def test_oracle_matcher_matches_reference(exp_golden, monkeypatch):
    """The oracle's match_eigenvectors (the checker of the device matcher)
    reproduces the reference's sigma/theta on the dense solutions."""
    monkeypatch.setattr(sequence, "_b_is_hpd", _host_hpd)
    for name, sp in _specs(exp_golden):
        sched = pkg.CorrelationSchedule(**sp["schedule"])
        blk = int(exp_golden[f"{name}/blk"])
        tracked = max(1, int(np.ceil(sp["fraction"] * sp["nev"])))
        vecs = []
        for _, a, b in sequence.iter_generated_sequence(sp["n"], sched, sp["seed"]):
            h, _ = orc.to_standard(a, b)
            vecs.append(np.linalg.eigh(h)[1][:, : max(blk + 1, sp["nev"])][:, :tracked])
        for i in range(len(vecs) - 1):
            sigma, theta = orc.match_eigenvectors(vecs[i], vecs[i + 1])
            np.testing.assert_array_equal(sigma, exp_golden[f"{name}/sigma/{i + 1}"])
            np.testing.assert_allclose(theta, exp_golden[f"{name}/theta/{i + 1}"], rtol=1e-6,
                                       atol=1e-9)


def test_payload_policy():
    a = np.zeros((2, 2))
    t = torch.zeros(2, 2)
    assert _device.get_array_output() == "auto"
    assert _device.host_output(a, None) and not _device.host_output(a, t)
    with _device.array_output("torch"):
        assert not _device.host_output(a)
    with _device.array_output("numpy"):
        assert _device.host_output(t)
    assert _device.host_output(a)
    with pytest.raises(ValueError):
        _device.set_array_output("cupy")
    assert isinstance(_device.emit(t, True), np.ndarray) and _device.emit(t, False) is t
