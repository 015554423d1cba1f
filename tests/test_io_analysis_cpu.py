"""Binary pencil I/O (row f2) and the host half of the angle report (row f4), CPU only."""

import json

import numpy as np
import pytest
import scipy.io

from paper_1206_3768_b200.analysis import greedy_match
from paper_1206_3768_b200.pencil_io import FormatError, load_sequence, read_pencil, save_sequence
from paper_1206_3768_b200.sequence import iter_baseline_sequence
from tests.golden.recipes import random_hermitian, random_spd


def test_npy_sequence_round_trip_is_bit_exact(tmp_path):
    seq = list(iter_baseline_sequence(40, 4, seed=3))
    man = save_sequence(seq, tmp_path, provenance={"kind": "generated", "seed": 3})
    assert man["n"] == 40 and man["length"] == 4 and man["format"] == "npy"
    assert json.load(open(tmp_path / "manifest.json"))["provenance"]["seed"] == 3
    back = load_sequence(tmp_path)
    assert [lab for lab, _, _ in back] == [1, 2, 3, 4]
    for (la, a, b), (lb, a2, b2) in zip(seq, back):
        assert la == lb and np.array_equal(a, a2) and np.array_equal(b, b2)


def test_reads_reference_matrix_market_directory(tmp_path):
    """The reference writes A_<l>.mtx / B_<l>.mtx (complex hermitian, 17
    digits) plus manifest.json (pencil_io.py:41-42, 86-98)."""
    rng = np.random.default_rng(5)
    a, b = random_hermitian(rng, 12), random_spd(rng, 12)
    for name, m in (("A", a), ("B", b)):
        scipy.io.mmwrite(str(tmp_path / f"{name}_1.mtx"), m, field="complex", symmetry="hermitian",
                         precision=17)
    json.dump({"n": 12, "length": 1, "provenance": {}}, open(tmp_path / "manifest.json", "w"))
    (lab, a2, b2), = load_sequence(tmp_path)
    assert lab == 1 and np.array_equal(a2, a) and np.array_equal(b2, b)


def test_format_errors(tmp_path):
    with pytest.raises(FormatError):
        load_sequence(tmp_path)  # no manifest
    json.dump({"n": 4, "length": 1}, open(tmp_path / "manifest.json", "w"))
    with pytest.raises(FormatError):
        load_sequence(tmp_path)  # no matrices
    np.save(tmp_path / "A_1.npy", np.zeros((4, 3), complex))
    np.save(tmp_path / "B_1.npy", np.zeros((4, 4), complex))
    with pytest.raises(FormatError):
        read_pencil(tmp_path, 1)
    with pytest.raises(FormatError):
        save_sequence([(2, np.eye(3, dtype=complex), np.eye(3, dtype=complex))], tmp_path / "x")


def reference_greedy(gram):
    """The reference's loop (sequence.py:209-216), restated for the check."""
    work = gram.copy()
    m = gram.shape[0]
    sigma = np.full(m, -1, dtype=int)
    for _ in range(m):
        i, j = np.unravel_index(np.argmax(work), work.shape)
        sigma[i] = j
        work[i, :] = -1.0
        work[:, j] = -1.0
    return sigma


@pytest.mark.parametrize("m,seed,ties", [(1, 0, False), (7, 1, False), (40, 2, False),
                                         (25, 3, True), (120, 4, True)])
def test_greedy_matching_equals_reference_loop(m, seed, ties):
    rng = np.random.default_rng(seed)
    gram = np.abs(rng.standard_normal((m, m)))
    gram += 3 * np.eye(m)[rng.permutation(m)]
    if ties:
        gram = np.round(gram, 1)  # many equal entries: tie order must match argmax's
    assert np.array_equal(greedy_match(gram), reference_greedy(gram))


def test_host_block_draw_is_bitwise_the_oracle_draw():
    """The solver's start/repair block draw (two float draws written into
    complex storage) gives the oracle's `re + 1j*im` bytes and leaves the
    generator in the same state (chfsi.py:323, _util.py:15-18)."""
    from oracle.chfsi_oracle import random_block
    from paper_1206_3768_b200.chfsi import _draw_block

    for n, cols in ((1, 1), (37, 5), (512, 48)):
        r1, r2 = np.random.default_rng((0, n, 0)), np.random.default_rng((0, n, 0))
        got = _draw_block(r1, n, cols).numpy()
        want = np.ascontiguousarray(random_block(r2, n, cols))
        assert got.shape == (n, cols)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
        assert r1.standard_normal() == r2.standard_normal()
