"""Reference basis files (mbstate.py:242-267) and the reference grouping
(group_orbitals, pipeline.py:123-159) on the host — CPU tests; the device
build from a file is pinned in test_gpu_parity.py."""
import json

import numpy as np
import pytest

from golden_util import GOLDEN, load_fixture

import paper_2110_10765_b200 as pkg

NAMES = ("skel_small", "skel_n1024", "skel_identity")


@pytest.mark.parametrize("name", NAMES)
def test_load_and_group_matches_reference_basis(name):
    """A basis file written by the reference's save_basis, loaded and grouped
    here, gives exactly the reference's grouped Basis arrays (occ_mat,
    bits_lo) that built the fixture's skeleton."""
    meta = json.loads((GOLDEN / "basis_files.json").read_text())[name]
    occ, lo, n_sp = pkg.load_basis(GOLDEN / f"basis_{name}.txt")
    f = load_fixture(f"{name}.npz")
    assert n_sp == int(f["basis_n_sp"]) and occ.shape == f["basis_occ"].shape
    g_occ, g_lo, perm, starts = pkg.group_basis(occ, lo, meta["group_bits"])
    assert np.array_equal(g_occ, f["basis_occ"])
    assert np.array_equal(g_lo, f["basis_bits_lo"])
    assert np.array_equal(occ[perm], g_occ)
    # orbital starts = the fixture's orbital table (id, start, stop)
    assert np.array_equal(starts, f["orb"][:, 1])


def test_save_load_round_trip(tmp_path):
    occ = np.array([[1, 2, 70], [3, 64, 65], [2, 5, 128]], np.uint16)
    p = tmp_path / "b.txt"
    pkg.save_basis(p, occ, 128)
    occ2, lo, n_sp = pkg.load_basis(p)
    assert n_sp == 128 and np.array_equal(occ, occ2)
    assert lo.tolist() == [3, (1 << 2) | (1 << 63), (1 << 1) | (1 << 4)]


@pytest.mark.parametrize("text,msg", [
    ("", "empty basis file"),
    ("6\n1 2 3 4 5 6\n", "malformed header"),
    ("3 128\n1 2 x\n", "malformed state line"),
    ("3 128\n", "no states after header"),
    ("3 128\n1 2 3\n1 2 3\n", "duplicate state"),
    ("3 128\n1 2 3\n1 2\n", "basis requires 3"),
    ("3 128\n1 2 129\n", "out of range"),
    ("3 128\n1 3 2\n", "strictly increasing"),
    ("3 128\n0 1 2\n", "1-based"),
])
def test_load_basis_errors(tmp_path, text, msg):
    """The reference's validation and messages (mbstate.py:93-118, :136-157, :249-267)."""
    p = tmp_path / "bad.txt"
    p.write_text(text)
    with pytest.raises(ValueError, match=msg):
        pkg.load_basis(p)


def test_group_bits_range():
    occ = np.array([[1, 2]], np.uint16)
    with pytest.raises(ValueError):
        pkg.group_basis(occ, np.array([3], np.uint64), 0)
