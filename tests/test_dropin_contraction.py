"""The reference's TestContraction (pkg/tests/test_pipeline.py:244-305) run
against the GPU package with only the import swapped.

``contract_observables`` / ``contract_oracle`` here take the reference's
exact arguments — a list of orbital ``Tile``s, the ``Orbital``s, the grouped
basis and the ``InteractionRank`` (pipeline.py:534-589).  The bases are the
ones the reference's ``random_basis`` produced for those tests, recorded by
tests/golden/make_golden.py (``contraction_cases.npz``) together with the
reference's own grouping, tile list and contraction outputs, so besides the
test bodies' own gates the GPU results are compared with the reference's
numbers.  The CPU tests pin the host helpers (grouping, tile enumeration)
and the validation order; the GPU tests need the device.
"""

import numpy as np
import pytest
import torch

from golden_util import load_fixture

import paper_2110_10765_b200 as pkg
from paper_2110_10765_b200 import (
    BasisArrays,
    InteractionRank,
    ObservablesInput,
    contract_observables,
    contract_oracle,
    enumerate_tiles,
    group_orbitals,
    random_coefficients,
)

CASES = load_fixture("contraction_cases.npz")
_BASES = {(64, 13): "p64", (128, 13): "p128", (256, 17): "p256"}


def random_basis(n, particles, bias=0.0, seed=0):
    """Stand-in for mbstate.random_basis: the reference's output for the
    tests' arguments, from the fixture (basis generation is out of scope)."""
    name = _BASES[(n, seed)]
    occ = CASES[f"{name}_occ"]
    assert occ.shape == (n, particles)
    return BasisArrays(occ, CASES[f"{name}_bits_lo"], int(CASES[f"{name}_n_sp"]))


class _Counts:
    def __init__(self, total):
        self.total = int(total)


def count_pairs(grouped, _grouped, rank):
    """Stand-in for sparsity.count_pairs(...).total: the reference's count
    for the fixture basis (the device build reproduces it, see
    test_pair_count_matches_reference)."""
    for name in ("p64", "p128", "p256"):
        if grouped.occ_mat.shape == CASES[f"{name}_grouped_occ"].shape and np.array_equal(
                grouped.occ_mat, CASES[f"{name}_grouped_occ"]):
            return _Counts(CASES[f"{name}_n_pairs"])
    raise KeyError("basis not in the fixture")


def contraction_tolerance(c: np.ndarray, n_pairs: int) -> float:  # test_pipeline.py:33-36
    return 2.0 ** -20 * max(n_pairs, 1) * float(np.abs(c).max()) ** 2


def small_problem(n=192, seed=13, group_bits=8):  # test_pipeline.py:39-44
    basis = random_basis(n, 6, bias=0.2, seed=seed)
    grouped, orbitals = group_orbitals(basis, group_bits=group_bits)
    rank = InteractionRank()
    tiles = enumerate_tiles(orbitals, orbitals, rank)
    return grouped, orbitals, tiles, rank


# ----------------------------------------------------------------------------
# CPU: host helpers and validation order
# ----------------------------------------------------------------------------

@pytest.mark.parametrize("name,n,seed,particles", [("p64", 64, 13, 6), ("p128", 128, 13, 6), ("p256", 256, 17, 8)])
def test_grouping_and_tiles_match_reference(name, n, seed, particles):
    """group_orbitals / enumerate_tiles reproduce the reference's state order,
    orbitals (id, start, stop, key) and tile list exactly."""
    grouped, orbs = group_orbitals(random_basis(n, particles, seed=seed), group_bits=int(CASES[f"{name}_group_bits"]))
    assert np.array_equal(grouped.occ_mat, CASES[f"{name}_grouped_occ"])
    got = np.array([(o.id, o.start, o.stop, o.key) for o in orbs], np.int64)
    assert np.array_equal(got, CASES[f"{name}_orb"])
    tiles = enumerate_tiles(orbs, orbs, InteractionRank())
    assert np.array_equal(np.array([(t.row_orbital, t.col_orbital) for t in tiles], np.int64), CASES[f"{name}_tiles"])


def test_input_validation():  # test_pipeline.py:293-299
    with pytest.raises(ValueError):
        ObservablesInput(c=np.zeros(4, dtype=np.float32), m_ops=1)
    with pytest.raises(ValueError):
        ObservablesInput(c=np.zeros((2, 4), dtype=np.float32), m_ops=0)
    with pytest.raises(ValueError):
        ObservablesInput(c=np.zeros((2, 4), dtype=np.float32), m_ops=1, op_kind="dense")


def test_accum_layout():  # test_pipeline.py:288-291
    inputs = ObservablesInput(c=np.zeros((3, 8), dtype=np.float32), m_ops=5)
    assert inputs.accum.shape == (15,)
    assert inputs.n_vec == 3


def test_coefficient_basis_size_checked():  # test_pipeline.py:301-305 (raises before any device work)
    grouped, orbs, tiles, rank = small_problem(n=64)
    inputs = ObservablesInput(c=np.zeros((2, 50), dtype=np.float32), m_ops=1)
    with pytest.raises(ValueError):
        contract_observables(tiles, orbs, grouped, rank, inputs)


def test_unknown_orbital_id_raises_keyerror():
    """A Tile naming an orbital that is not in the list fails like the
    reference's orb_by_id lookup (pipeline.py:436-443)."""
    from paper_2110_10765_b200 import Tile
    from paper_2110_10765_b200.observables import _tile_ranges

    grouped, orbs, tiles, rank = small_problem(n=64)
    with pytest.raises(KeyError):
        _tile_ranges(list(tiles) + [Tile(10_000, orbs[0].id)], orbs, False)
    r = _tile_ranges(tiles, orbs, True)
    f = _tile_ranges(tiles, orbs, False)
    assert np.array_equal(r[:, :2], f[:, 2:]) and np.array_equal(r[:, 2:], f[:, :2])


def test_validation_order_and_messages():
    """pipeline.py:550-555: strategy first, then the coefficient size; then
    the worker count (resolve_workers, _util.py:41-42)."""
    grouped, orbs, tiles, rank = small_problem(n=64)
    bad = ObservablesInput(c=np.zeros((2, 50), dtype=np.float32), m_ops=1)
    with pytest.raises(ValueError, match="unknown strategy 'nope'"):
        contract_observables(tiles, orbs, grouped, rank, bad, "nope")
    with pytest.raises(ValueError, match="coefficients cover 50 states, basis has 64"):
        contract_observables(tiles, orbs, grouped, rank, bad)
    ok = ObservablesInput(c=np.zeros((2, 64), dtype=np.float32), m_ops=1)
    with pytest.raises(ValueError, match="workers must be >= 1"):
        contract_observables(tiles, orbs, grouped, rank, ok, workers=0)
    with pytest.raises(ValueError):
        contract_oracle(tiles, orbs, grouped, rank, bad)


# ----------------------------------------------------------------------------
# GPU: the TestContraction bodies, plus the reference's recorded outputs
# ----------------------------------------------------------------------------

gpu = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=False)
def device():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    pkg.lib()
    return torch.device("cuda", 0)


@gpu
def test_zero_vectors_zero_accum(device):  # test_pipeline.py:245-249
    grouped, orbs, tiles, rank = small_problem(n=64)
    inputs = ObservablesInput(c=np.zeros((4, 64), dtype=np.float32), m_ops=3)
    out = contract_observables(tiles, orbs, grouped, rank, inputs)
    assert not out.any()


@gpu
def test_identity_operator_unit_vectors(device):  # test_pipeline.py:251-264
    # ±n**-0.5 entries at n = 4**k make float32 sums of squares exact
    n = 256
    basis = random_basis(n, 8, bias=0.1, seed=17)
    grouped, orbs = group_orbitals(basis, group_bits=8)
    rank = InteractionRank()
    tiles = enumerate_tiles(orbs, orbs, rank)
    inputs = ObservablesInput(
        c=random_coefficients(4, n, seed=1, kind="signs"),
        m_ops=3,
        op_kind="identity",
    )
    out = contract_observables(tiles, orbs, grouped, rank, inputs)
    assert np.all(np.abs(out - 1.0) <= 2.0 ** -20)


@gpu
@pytest.mark.parametrize("strategy", ["array_clause", "atomic_per_element", "generated_scalars"])
def test_strategies_match_oracle(device, strategy):  # test_pipeline.py:266-276
    grouped, orbs, tiles, rank = small_problem(n=128)
    inputs = ObservablesInput(
        c=random_coefficients(4, 128, seed=2), m_ops=3, seed=4
    )
    got = contract_observables(tiles, orbs, grouped, rank, inputs, strategy)
    want = contract_oracle(tiles, orbs, grouped, rank, inputs)
    n_pairs = count_pairs(grouped, grouped, rank).total
    tol = contraction_tolerance(inputs.c, n_pairs)
    assert np.abs(got.astype(np.float64) - want).max() <= tol
    # and against the reference's own numbers for the same call
    assert np.abs(got.astype(np.float64) - CASES[f"strat_{strategy}"]).max() <= tol
    assert np.abs(want - CASES["strat_oracle"]).max() <= 1e-12 * max(1.0, np.abs(want).max())
    # the returned array is a view of inputs.accum, filled in place (pipeline.py:569-570)
    assert np.shares_memory(got, inputs.accum) and got.shape == (4, 3)


@gpu
def test_hermitian_symmetry(device):  # test_pipeline.py:278-286
    grouped, orbs, tiles, rank = small_problem(n=128)
    c = random_coefficients(4, 128, seed=3)
    fwd = ObservablesInput(c=c, m_ops=2, seed=6)
    rev = ObservablesInput(c=c, m_ops=2, seed=6)
    a = contract_observables(tiles, orbs, grouped, rank, fwd).copy()
    b = contract_observables(tiles, orbs, grouped, rank, rev, transpose=True).copy()
    n_pairs = count_pairs(grouped, grouped, rank).total
    assert np.abs(a - b).max() <= contraction_tolerance(c, n_pairs)
    assert np.abs(a - CASES["herm_fwd"]).max() <= contraction_tolerance(c, n_pairs)
    assert np.abs(b - CASES["herm_rev"]).max() <= contraction_tolerance(c, n_pairs)


@gpu
@pytest.mark.parametrize("name", ["skel_small.npz", "skel_n1024.npz", "skel_identity.npz"])
def test_skeleton_fixtures_through_reference_signature(device, name):
    """The three skeleton fixtures (n = 192 / 1024 / 1024-identity) through
    the reference signature, from their recorded grouped basis, orbitals and
    tiles: the reference's contract_observables (forward, transposed) and
    contract_oracle numbers."""
    f = load_fixture(name)
    from paper_2110_10765_b200 import Orbital, Tile

    grouped = BasisArrays(f["basis_occ"], f["basis_bits_lo"], int(f["basis_n_sp"]))
    orbs = [Orbital(id=int(a), key=None, start=int(b), stop=int(c)) for a, b, c in f["orb"]]
    tiles = [Tile(int(r), int(c)) for r, c, _, _ in f["tiles_rc"]]
    rank = InteractionRank(d=int(f["rank_threshold"]) // 2)
    c = f["X"].T.copy()
    mk = lambda: ObservablesInput(c=c, m_ops=int(f["m_ops"]), op_kind=str(f["op_kind"]), seed=int(f["op_seed"]))  # noqa: E731
    tol = contraction_tolerance(c, int(f["nnz"]))
    got = contract_observables(tiles, orbs, grouped, rank, mk()).astype(np.float64)
    assert np.abs(got - f["accum"]).max() <= tol
    got_t = contract_observables(tiles, orbs, grouped, rank, mk(), transpose=True).astype(np.float64)
    assert np.abs(got_t - f["accum_transpose"]).max() <= tol
    want = contract_oracle(tiles, orbs, grouped, rank, mk())
    assert np.abs(want - f["accum_oracle"]).max() <= 1e-12 * max(1.0, np.abs(f["accum_oracle"]).max())


@gpu
def test_tile_subset_and_many_vectors(device):
    """A tile list that is NOT the full enumeration (every third tile, so
    the pair set is not symmetric) and vector / operator counts beyond one
    8 × 8 chunk: the device walk equals the f64 numpy restatement over the
    same explicit pairs (oracle.contract_vmv)."""
    from oracle import oracle

    grouped, orbs, tiles, rank = small_problem(n=128)
    sub = tiles[::3]
    ob = {o.id: o for o in orbs}
    occ, lo = grouped.occ_mat, grouped.bits_lo
    I, J = [], []
    for t in sub:
        r, q = ob[t.row_orbital], ob[t.col_orbital]
        for i in range(r.start, r.stop):
            for j in range(q.start, q.stop):
                if bin(int(lo[i]) ^ int(lo[j])).count("1") <= rank.threshold and \
                        oracle.occ_diff(occ[i], occ[j]) <= rank.threshold:
                    I.append(i)
                    J.append(j)
    I, J = np.array(I), np.array(J)
    c = random_coefficients(11, 128, seed=5)
    inp = ObservablesInput(c=c, m_ops=10, seed=3)
    got = contract_observables(sub, orbs, grouped, rank, inp).astype(np.float64)
    want = oracle.contract_vmv(c, I, J, 10, 1, 3)
    assert np.abs(got - want).max() <= contraction_tolerance(c, I.size)
    exact = contract_oracle(sub, orbs, grouped, rank, ObservablesInput(c=c, m_ops=10, seed=3))
    assert np.abs(exact - want).max() <= 1e-12 * max(1.0, np.abs(want).max())


@gpu
@pytest.mark.parametrize("name,n,seed,particles", [("p64", 64, 13, 6), ("p128", 128, 13, 6), ("p256", 256, 17, 8)])
def test_pair_count_matches_reference(device, name, n, seed, particles):
    """The device build of the fixture basis holds exactly the reference's
    count_pairs(...).total interacting pairs (both triangles; the stand-in
    count_pairs above returns the recorded number)."""
    grouped, _ = group_orbitals(random_basis(n, particles, seed=seed), group_bits=int(CASES[f"{name}_group_bits"]))
    H = pkg.HalfTiles.from_basis(grouped, rank=InteractionRank())
    rc, tiles = H.export_dense()
    nz = tiles != 0
    per_tile = nz.reshape(nz.shape[0], -1).sum(1)
    full = int(per_tile[rc[:, 0] == rc[:, 1]].sum() + 2 * per_tile[rc[:, 0] != rc[:, 1]].sum())
    assert full == int(CASES[f"{name}_n_pairs"])
