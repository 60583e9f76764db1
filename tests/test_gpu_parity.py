"""GPU parity: the sm_100a path through the C-ABI vs the CPU oracle.

Gate (BASELINE.json north star): ‖ΔY‖_F / (‖A‖_F·‖X‖_F) ≤ 1e-5 (f32),
≤ 1e-12 (f64); plus the componentwise bound |ΔY| ≤ (c+2)·u·(|A||X|) with
c = max row nnz, u = 2⁻²⁴ (f32) / 2⁻⁵³ (f64), which a TF32 shortcut fails.
Structure and values are bit-exact (integer/bitwise comparisons).
"""

import json
import os

import numpy as np
import pytest
import torch

from golden_util import GOLDEN, load_fixture
from oracle import oracle

pytestmark = pytest.mark.gpu

F32_GATE, F64_GATE = 1e-5, 1e-12
U32, U64 = 2.0 ** -24, 2.0 ** -53


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2110_10765_b200 as p

    return p


def check_result(n, rc, tiles, X, Y, dtype):
    """Normwise + componentwise gates against the f64 oracle."""
    X = np.asarray(X, np.float64)
    Y_ref = oracle.sym_spmm(n, rc, tiles, X)
    A_f = oracle.frobenius_full(rc, tiles)
    err = oracle.normwise_error(Y, Y_ref, A_f, X)
    gate = F32_GATE if dtype == torch.float32 else F64_GATE
    assert err <= gate, f"normwise error {err:.3e} > {gate}"
    u = U32 if dtype == torch.float32 else U64
    nnz_row = 64 * max(1, int(np.bincount(np.concatenate([rc[:, 0], rc[rc[:, 0] != rc[:, 1], 1]])).max()))
    absAX = oracle.abs_product(n, rc, tiles, X)
    assert oracle.componentwise_ok(Y, Y_ref, absAX, nnz_row, u), "componentwise bound violated"
    return err


def f32bits(a):
    return np.asarray(a, dtype=np.float32).view(np.uint32)


# ----------------------------------------------------------------------------
# device hash / value generation / repacking: bit-exact
# ----------------------------------------------------------------------------

def test_device_hash_matches_reference_kats(pkg):
    kat = json.loads((GOLDEN / "hash_kat.json").read_text())
    for key, kind in (("h", 0), ("op", None)):
        cases = kat[key]
        I = torch.tensor([c["i"] for c in cases], dtype=torch.int64, device="cuda")
        J = torch.tensor([c["j"] for c in cases], dtype=torch.int64, device="cuda")
        for idx, c in enumerate(cases):
            kd = kind if kind is not None else (1 if c["op_code"] == 1 else 2)
            out = torch.empty(1, dtype=torch.float32, device="cuda")
            pkg._lib.check(pkg.lib().cim_hash_values(I[idx:].data_ptr(), J[idx:].data_ptr(), 1, kd, c["seed"],
                                                     c.get("k", 0), out.data_ptr(), None), "hash")
            torch.cuda.synchronize()
            assert int(f32bits(out.cpu().numpy())[0]) == c["bits"], c


F32_LAYOUTS = ["tc", "frag"]
DT_LAYOUTS = [(torch.float32, "tc"), (torch.float32, "frag"), (torch.float64, "frag"), (torch.float64, "tc")]


@pytest.mark.parametrize("dtype,layout", DT_LAYOUTS)
@pytest.mark.parametrize("values,kind", [("h_xor", 0), ("op_hash", 1), ("identity", 2)])
def test_synthetic_values_bit_exact(pkg, dtype, layout, values, kind):
    n = 1000  # ragged: last block half empty
    rc = pkg.synthetic_pattern((n + 63) // 64, 0.3, seed=1)
    H = pkg.HalfTiles.synthetic(n, tile_rc=rc, values=values, value_seed=7, op_k=2, dtype=dtype, layout=layout)
    got = H.dense_tiles().cpu().numpy()
    want = oracle.synthetic_dense_tiles(n, rc, seed=7, kind=kind, op_k=2).astype(got.dtype)
    assert np.array_equal(got.view(np.uint8), want.view(np.uint8))


@pytest.mark.parametrize("dtype,layout", DT_LAYOUTS)
def test_pack_matches_host_layout_and_roundtrips(pkg, dtype, layout):
    from paper_2110_10765_b200.halftiles import fragment_pack_host

    rng = np.random.default_rng(3)
    npd = np.float32 if dtype == torch.float32 else np.float64
    tiles = rng.standard_normal((5, 64, 64)).astype(npd)
    rc = np.array([[0, 0], [0, 2], [1, 1], [1, 3], [2, 2]], np.int32)
    H = pkg.HalfTiles.from_dense_tiles(4 * 64, rc, tiles, dtype=dtype, layout=layout)
    assert np.array_equal(H.vals.cpu().numpy(), fragment_pack_host(tiles, layout))
    assert np.array_equal(H.dense_tiles().cpu().numpy(), tiles)


# ----------------------------------------------------------------------------
# SpMM parity on reference skeletons
# ----------------------------------------------------------------------------

@pytest.mark.parametrize("name", ["skel_small.npz", "skel_n1024.npz", "skel_identity.npz"])
@pytest.mark.parametrize("dtype,layout", DT_LAYOUTS)
def test_reference_skeleton_spmm(pkg, name, dtype, layout):
    f = load_fixture(name)
    n = int(f["n"])
    from paper_2110_10765_b200.halftiles import dense_break_even
    H = pkg.HalfTiles.from_coo(n, f["i"], f["j"], f["v"], dtype=dtype, layout=layout,
                               dense_fill=dense_break_even(dtype))
    # ragged orbital blocks: most 64-tiles fall below the memory break-even → sparse tiles
    if name == "skel_n1024.npz":
        assert H.n_sparse_tiles > H.n_tiles
    # structure: the stored half-tile set reproduces the reference pair set exactly
    rc, tiles = H.export_dense()
    i, j, v = oracle.half_tiles_to_coo(n, rc, tiles)
    assert oracle.pair_set_digest(i, j) == str(f["pair_digest"])
    X = torch.from_numpy(f["X"]).to(dtype)
    Y = pkg.sym_spmm(H, X.cuda()).cpu().numpy()
    check_result(n, rc, tiles.astype(np.float64), f["X"], Y, dtype)
    # against the reference's matrix product computed by scipy from its COO
    rel = np.linalg.norm(Y - f["Y_ref"]) / np.linalg.norm(f["Y_ref"])
    assert rel <= (1e-5 if dtype == torch.float32 else 1e-12)


@pytest.mark.parametrize("name", ["skel_small.npz", "skel_n1024.npz", "skel_identity.npz"])
@pytest.mark.parametrize("layout", F32_LAYOUTS)
def test_contract_observables_matches_reference(pkg, name, layout):
    f = load_fixture(name)
    n = int(f["n"])
    pattern = pkg.HalfTiles.from_coo(n, f["i"], f["j"], np.ones_like(f["v"]), layout=layout)
    c = f["X"].T.copy()
    inp = pkg.ObservablesInput(c=c, m_ops=int(f["m_ops"]), op_kind=str(f["op_kind"]), seed=int(f["op_seed"]))
    got = pkg.contract_pattern(pattern, inp).astype(np.float64)
    tol = oracle.contraction_tolerance(c, int(f["nnz"]))
    assert np.abs(got - f["accum_oracle"]).max() <= tol
    assert np.abs(got - f["accum"]).max() <= tol
    got_t = pkg.contract_pattern(pattern, pkg.ObservablesInput(c=c, m_ops=int(f["m_ops"]),
                                                                  op_kind=str(f["op_kind"]), seed=int(f["op_seed"])),
                                     transpose=True)
    assert np.abs(got_t - got).max() <= tol
    if str(f["op_kind"]) == "identity":
        assert np.all(np.abs(got - 1.0) <= 2.0 ** -20)


@pytest.mark.parametrize("dtype,layout", [(torch.float32, "frag"), (torch.float32, "tc"), (torch.float64, "frag"),
                                          (torch.float64, "tc")])
@pytest.mark.parametrize("n_vec,m_ops,op_kind", [(1, 1, "symmetric_hash"), (8, 3, "symmetric_hash"),
                                                 (16, 16, "symmetric_hash"), (5, 7, "identity"),
                                                 (20, 19, "symmetric_hash")])
def test_contract_fused_vs_oracle(pkg, dtype, layout, n_vec, m_ops, op_kind):
    """cim_contract_observables (O_ij(k) on the fly, one tile walk) on a
    ragged pattern with dense and sparse tiles: matches the f64 oracle
    contract_vmv over the full pair list within the reference tolerance, and
    the materialised composition (fill O_k + sym_spmm + dot); vector and
    operator counts beyond one chunk (16) exercise the host chunk loops."""
    rng = np.random.default_rng(n_vec * 31 + m_ops)
    n = 1000
    nb = (n + 63) // 64
    rc = pkg.synthetic_pattern(nb, 0.3, seed=3)
    ii, jj = [], []
    for t, (R, C) in enumerate(rc):
        fill = 0.9 if t % 3 == 0 else 0.02
        m = rng.random((64, 64)) < fill
        if R == C:
            m = m | m.T
        a, b = np.nonzero(m)
        ii.append(R * 64 + a)
        jj.append(C * 64 + b)
    i = np.concatenate(ii)
    j = np.concatenate(jj)
    ok = (i < n) & (j < n)
    key = np.unique(np.minimum(i[ok], j[ok]) * n + np.maximum(i[ok], j[ok]))
    lo, hi = key // n, key % n
    I = np.concatenate([lo, hi[lo != hi]])
    J = np.concatenate([hi, lo[lo != hi]])
    pattern = pkg.HalfTiles.from_coo(n, I, J, np.ones(I.size), dtype=dtype, layout=layout)
    if layout == "frag":
        assert pattern.n_sparse_tiles > 0 and pattern.n_tiles > 0
    c = pkg.random_coefficients(n_vec, n, seed=n_vec, kind="gauss")
    seed = 11
    inp = pkg.ObservablesInput(c=c, m_ops=m_ops, op_kind=op_kind, seed=seed)
    got = pkg.contract_pattern(pattern, inp).astype(np.float64)
    code = {"symmetric_hash": 1, "identity": 2}[op_kind]  # C ABI (CIM_VALUES_*)
    want = oracle.contract_vmv(c, I, J, m_ops, {"symmetric_hash": 1, "identity": 0}[op_kind], seed)
    tol = oracle.contraction_tolerance(c, I.size)
    assert np.abs(got - want).max() <= tol
    from paper_2110_10765_b200.observables import contract_materialized
    mat = contract_materialized(pattern, inp)  # every width: sparse tiles too wide for the ring run as passes
    assert np.abs(got - mat).max() <= tol
    # accumulate flag through the C ABI: a second walk doubles the result
    dev_c = torch.from_numpy(c).cuda().t().contiguous()
    acc = torch.zeros((n_vec, m_ops), dtype=torch.float64, device="cuda")
    L = pkg._lib.lib()
    for _ in range(2):
        assert L.cim_contract_observables(pattern.descriptor(), dev_c.data_ptr(), n_vec, m_ops, code, seed,
                                          acc.data_ptr(), 1, None) == 0
    assert np.abs(acc.cpu().numpy() - 2 * got).max() <= 2 * tol


@pytest.mark.parametrize("layout", F32_LAYOUTS)
def test_single_state_diagonal(pkg, layout):
    # test_pipeline.py:131-138: one state → nnz 1, stored value exactly h(0,0,0)
    h0 = np.array([oracle.h_values(0, 0, 0)], np.float32).reshape(1)
    H = pkg.HalfTiles.from_coo(1, [0], [0], h0, layout=layout, dense_fill=0.0)
    assert H.n_tiles == 1 and H.n == 1
    assert H.dense_tiles()[0, 0, 0].item() == float(h0[0])
    Y = pkg.sym_spmm(H, torch.tensor([[2.0]], device="cuda"))
    want = 2.0 * float(h0[0])
    if layout == "frag":
        assert float(Y[0, 0]) == want  # one FFMA: exact
    else:
        assert abs(float(Y[0, 0]) - want) <= 2.0 ** -19 * abs(want)  # split-TF32 residual


# ----------------------------------------------------------------------------
# synthetic configs, vector-count sweep, edge cases
# ----------------------------------------------------------------------------

@pytest.fixture(scope="module")
def c1_small(pkg):
    """A C1-family matrix (block 64, Bernoulli tiles) small enough for the f64
    numpy oracle: n = 8192 - 37 (ragged), p = 0.05."""
    n = 8192 - 37
    rc = pkg.synthetic_pattern((n + 63) // 64, 0.05, seed=11)
    tiles = oracle.synthetic_dense_tiles(n, rc, seed=0)
    return n, rc, tiles


@pytest.mark.parametrize("layout", F32_LAYOUTS)
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 7, 8, 9, 16, 24, 32, 40, 48, 56, 63, 64])
def test_k_sweep_f32(pkg, c1_small, k, layout):
    n, rc, tiles = c1_small
    H = pkg.HalfTiles.synthetic(n, tile_rc=rc, dtype=torch.float32, layout=layout)
    X = torch.randn((n, k), generator=torch.Generator().manual_seed(k))
    Y = pkg.sym_spmm(H, X.cuda()).cpu().numpy()
    check_result(n, rc, tiles, X.numpy(), Y, torch.float32)


@pytest.mark.parametrize("layout", ["frag", "tc"])
@pytest.mark.parametrize("k", [1, 2, 3, 4, 7, 8, 12, 16, 20, 24, 28, 32, 40, 44, 48, 60, 63, 64])
def test_k_sweep_f64(pkg, c1_small, k, layout):
    n, rc, tiles = c1_small
    H = pkg.HalfTiles.synthetic(n, tile_rc=rc, dtype=torch.float64, layout=layout)
    X = torch.randn((n, k), generator=torch.Generator().manual_seed(k), dtype=torch.float64)
    Y = pkg.sym_spmm(H, X.cuda()).cpu().numpy()
    check_result(n, rc, tiles.astype(np.float64), X.numpy(), Y, torch.float64)


@pytest.mark.parametrize("dtype,k,layout", [(torch.float32, 32, "frag"), (torch.float32, 64, "frag"),
                                             (torch.float64, 16, "frag"), (torch.float64, 64, "frag"),
                                             (torch.float32, 32, "tc"), (torch.float64, 64, "tc")])
def test_multipass_widths_on_concurrent_streams(pkg, c1_small, dtype, k, layout):
    """Widths above one pass stage a pass-major copy of X in a per-stream
    scratch buffer: applies queued on two streams at once (different X, same
    H) must each match their own oracle product, and repeated calls on one
    stream (the buffer reused) stay exact."""
    n, rc, tiles = c1_small
    H = pkg.HalfTiles.synthetic(n, tile_rc=rc, dtype=dtype, layout=layout)
    g = torch.Generator().manual_seed(k)
    Xs = [torch.randn((n, k), generator=g, dtype=dtype) for _ in range(2)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = []
    for X, st in zip(Xs, streams):
        with torch.cuda.stream(st):
            outs.append(pkg.sym_spmm(H, X.cuda(non_blocking=False), stream=st))
    torch.cuda.synchronize()
    tl = tiles if dtype == torch.float32 else tiles.astype(np.float64)
    for X, Y in zip(Xs, outs):
        check_result(n, rc, tl, X.numpy(), Y.cpu().numpy(), dtype)
    again = pkg.sym_spmm(H, Xs[0].cuda())
    assert (again - outs[0]).abs().max().item() <= 1e-5 * outs[0].abs().max().item()


@pytest.mark.parametrize("layout", F32_LAYOUTS)
def test_opaque_random_symmetric_values(pkg, c1_small, layout):
    """Values with no XOR structure (op hash of (min,max)) — the kernel must
    treat tile values as opaque streamed data (SURVEY.md §7 hard parts)."""
    n, rc, _ = c1_small
    H = pkg.HalfTiles.synthetic(n, tile_rc=rc, values="op_hash", value_seed=99, op_k=3, layout=layout)
    tiles = oracle.synthetic_dense_tiles(n, rc, seed=99, kind=1, op_k=3)
    X = torch.randn((n, 8), generator=torch.Generator().manual_seed(1))
    check_result(n, rc, tiles, X.numpy(), pkg.sym_spmm(H, X.cuda()).cpu().numpy(), torch.float32)


@pytest.mark.parametrize("layout", F32_LAYOUTS)
def test_c1_config_vs_c_oracle(pkg, layout):
    """BASELINE config 1: n=65,536, p=0.01 (5,244 off-diagonal tiles), k=8 f32."""
    from oracle import cpu

    n, k = 65536, 8
    H = pkg.HalfTiles.synthetic(n, p=0.01, seed=0, layout=layout)
    assert H.n_off_tiles == 5244 and H.n_diag_tiles == 1024
    rc = H.tile_rc_host
    tiles = cpu.fill_h(rc, n, 0)
    X = np.random.default_rng(0).standard_normal((n, k)).astype(np.float32)
    Y = pkg.sym_spmm(H, torch.from_numpy(X).cuda()).cpu().numpy()
    Y_ref = cpu.sym_spmm_f64(n, rc, tiles, X)
    err = oracle.normwise_error(Y, Y_ref, oracle.frobenius_full(rc, tiles), X)
    assert err <= F32_GATE
    # componentwise bound with |A||X|
    absAX = cpu.sym_spmm_f64(n, rc, np.abs(tiles), np.abs(X))
    nnz_row = 64 * int(np.bincount(np.concatenate([rc[:, 0], rc[rc[:, 0] != rc[:, 1], 1]])).max())
    assert oracle.componentwise_ok(Y, Y_ref, absAX, nnz_row, U32)


@pytest.mark.parametrize("dtype,layout,k", [(torch.float32, "tc", 4), (torch.float32, "frag", 4),
                                            (torch.float32, "tc", 32), (torch.float64, "frag", 4),
                                            (torch.float64, "tc", 16), (torch.float64, "tc", 64)])
@pytest.mark.parametrize("n", [1, 63, 64, 65, 200])
def test_ragged_and_tiny(pkg, n, dtype, layout, k):
    nb = (n + 63) // 64
    rc = pkg.synthetic_pattern(nb, 1.0, seed=0)  # every upper tile
    tiles = oracle.synthetic_dense_tiles(n, rc, seed=5)
    H = pkg.HalfTiles.synthetic(n, tile_rc=rc, value_seed=5, layout=layout, dtype=dtype)
    X = torch.randn((n, k), generator=torch.Generator().manual_seed(n), dtype=dtype)
    check_result(n, rc, tiles.astype(np.float64) if dtype == torch.float64 else tiles, X.numpy(),
                 pkg.sym_spmm(H, X.cuda(), layout="nk").cpu().numpy(), dtype)


@pytest.mark.parametrize("dtype,layout,k", [(torch.float32, "frag", 8), (torch.float32, "tc", 8),
                                            (torch.float32, "tc", 64), (torch.float64, "tc", 32),
                                            (torch.float64, "frag", 8)])
def test_diagonal_only_and_long_rows(pkg, dtype, layout, k):
    # no off-diagonal tiles at all; then a dense upper triangle (long block rows → many units)
    for p in (0.0, 1.0):
        n = 40 * 64
        rc = pkg.synthetic_pattern(40, p, seed=0)
        H = pkg.HalfTiles.synthetic(n, tile_rc=rc, max_unit=7, layout=layout, dtype=dtype)
        tiles = oracle.synthetic_dense_tiles(n, rc, seed=0)
        X = torch.randn((n, k), generator=torch.Generator().manual_seed(2), dtype=dtype)
        check_result(n, rc, tiles.astype(np.float64) if dtype == torch.float64 else tiles, X.numpy(),
                     pkg.sym_spmm(H, X.cuda()).cpu().numpy(), dtype)


def test_layouts_numpy_out_accumulate(pkg, c1_small):
    n, rc, tiles = c1_small
    H = pkg.HalfTiles.synthetic(n, tile_rc=rc)
    Xn = np.random.default_rng(4).standard_normal((n, 8)).astype(np.float32)
    Y_nk = pkg.sym_spmm(H, Xn)  # numpy in → numpy out
    assert isinstance(Y_nk, np.ndarray) and Y_nk.shape == (n, 8)
    Y_kn = pkg.sym_spmm(H, Xn.T.copy())  # reference (n_vec, n) layout
    assert Y_kn.shape == (8, n)
    assert np.abs(Y_kn.T - Y_nk).max() <= 1e-5 * np.abs(Y_nk).max()
    out = torch.ones((n, 8), device="cuda")
    pkg.sym_spmm(H, torch.from_numpy(Xn).cuda(), out=out, accumulate=True)
    assert np.abs(out.cpu().numpy() - (Y_nk + 1.0)).max() <= 1e-4 * np.abs(Y_nk).max()
    out2 = np.zeros((n, 8), np.float32)
    pkg.sym_spmm(H, Xn, out=out2)
    assert np.abs(out2 - Y_nk).max() <= 1e-5 * np.abs(Y_nk).max()


def test_validation_raises_before_compute(pkg, c1_small):
    n, rc, _ = c1_small
    H = pkg.HalfTiles.synthetic(n, tile_rc=rc)
    with pytest.raises(ValueError):
        pkg.sym_spmm(H, torch.zeros((n, 4), dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        pkg.sym_spmm(H, torch.zeros((n + 1, 4), device="cuda"))
    with pytest.raises(ValueError):
        pkg.sym_spmm(H, torch.zeros((n,), device="cuda"))
    with pytest.raises(ValueError):
        pkg.sym_spmm(H, torch.zeros((n, 4), device="cuda"), layout="xy")
    with pytest.raises(ValueError):
        pkg.HalfTiles.from_coo(4, [0, 1], [1, 0], np.array([1.0, 2.0], np.float32))  # not symmetric
    # the C-ABI itself rejects a strided X (ldx != k)
    X = torch.zeros((H.n_pad, 16), device="cuda")[:, :8]
    Y = torch.zeros((H.n_pad, 8), device="cuda")
    rc_ = pkg.lib().cim_sym_spmm(H.descriptor(), X.data_ptr(), Y.data_ptr(), 8, 16, 8, 0, None)
    assert rc_ == 1


def test_deterministic_structure_and_repeatable_values(pkg, c1_small):
    n, rc, _ = c1_small
    H1 = pkg.HalfTiles.synthetic(n, tile_rc=rc)
    H2 = pkg.HalfTiles.synthetic(n, tile_rc=rc)
    assert torch.equal(H1.vals, H2.vals)
    X = torch.randn((n, 8), generator=torch.Generator().manual_seed(0)).cuda()
    Ya, Yb = pkg.sym_spmm(H1, X), pkg.sym_spmm(H1, X)
    # float atomics: order-dependent only at the ulp level
    assert (Ya - Yb).abs().max().item() <= 1e-5 * Ya.abs().max().item()


def test_save_load_roundtrip(pkg, c1_small, tmp_path):
    n, rc, _ = c1_small
    H = pkg.HalfTiles.synthetic(n, tile_rc=rc)
    H.save(tmp_path / "h.npz")
    H2 = pkg.HalfTiles.load(tmp_path / "h.npz")
    assert torch.equal(H.vals, H2.vals) and np.array_equal(H.tile_rc_host, H2.tile_rc_host)
    # mixed dense + sparse storage round-trips too
    f = load_fixture("skel_n1024.npz")
    M = pkg.HalfTiles.from_coo(int(f["n"]), f["i"], f["j"], f["v"], dense_fill=0.5)
    M.save(tmp_path / "m.npz")
    M2 = pkg.HalfTiles.load(tmp_path / "m.npz")
    a, b = M.export_dense(), M2.export_dense()
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and M2.n_sparse_tiles == M.n_sparse_tiles


@pytest.mark.parametrize("dtype,k,layout", [(torch.float32, 8, "frag"), (torch.float32, 16, "tc"), (torch.float64, 8, "tc"),
                                             (torch.float32, 3, "frag"), (torch.float64, 12, "frag"),
                                             (torch.float32, 40, "tc"), (torch.float64, 20, "frag"),
                                             (torch.float64, 64, "tc")])
def test_sharded_world1_equals_direct(pkg, dtype, k, layout):
    n = 4000  # ragged: the last block row is partly padding
    S = pkg.ShardedSymSpmm.synthetic(n, k=k, p=0.1, seed=3, dtype=dtype, layout=layout)
    rc = pkg.synthetic_pattern((n + 63) // 64, 0.1, seed=3)
    H = pkg.HalfTiles.synthetic(n, tile_rc=rc, dtype=dtype, layout=layout)
    X = torch.zeros((S.rows_per_rank, k), dtype=dtype)  # the operator's rows: n_pad, rows ≥ n zero
    X[:n] = torch.randn((n, k), generator=torch.Generator().manual_seed(0), dtype=dtype)
    X = X.cuda()
    Y = S.apply(X)
    Yd = pkg.sym_spmm(H, X[:n].contiguous())
    assert torch.allclose(Y[:n], Yd, rtol=0, atol=1e-5 * Yd.abs().max().item())
    assert torch.all(Y[n:] == 0)


# ----------------------------------------------------------------------------
# BASELINE config 2 at full size: size-independent properties
# ----------------------------------------------------------------------------

@pytest.mark.slow
@pytest.mark.parametrize("layout", F32_LAYOUTS)
def test_c2_full_size_properties(pkg, layout):
    """n = 2²², ~2·10⁹ stored values, k = 8 f32 (8 GB in HBM).

    * symmetry:  ⟨X₁, A X₂⟩ = ⟨A X₁, X₂⟩   (every tile used both ways)
    * linearity: A(X₁ + 2X₂) = A X₁ + 2 A X₂
    * exact block rows: block row 0 and the last block row recomputed on the
      host from the oracle hash (row 0 has only direct tiles; the last row
      only its diagonal tile plus transposed contributions).
    """
    n, k = 1 << 22, 8
    nb = n // 64
    n_off = 488281 - 65536
    H = pkg.HalfTiles.synthetic(n, n_off=n_off, seed=0, layout=layout)
    assert abs(H.nnz_stored - 2_000_000_000) < 2_000_000 * 2
    g = torch.Generator(device="cuda").manual_seed(0)
    X1 = torch.randn((n, k), device="cuda", generator=g)
    X2 = torch.randn((n, k), device="cuda", generator=g)
    Y1 = pkg.sym_spmm(H, X1)
    Y2 = pkg.sym_spmm(H, X2)
    a = (X1.double() * Y2.double()).sum(0)
    b = (Y1.double() * X2.double()).sum(0)
    assert torch.all((a - b).abs() <= 1e-5 * (X1.double().abs() * Y2.double().abs()).sum(0))
    Y3 = pkg.sym_spmm(H, X1 + 2 * X2)
    lin = (Y3 - (Y1 + 2 * Y2)).norm() / (Y3.norm())
    assert lin.item() <= 1e-5
    rc = H.tile_rc_host
    X1h = X1.cpu().numpy()
    for R in (0, nb - 1):
        sel = np.flatnonzero((rc[:, 0] == R) | (rc[:, 1] == R))
        sub = rc[sel]
        tiles = oracle.synthetic_dense_tiles(n, sub, seed=0).astype(np.float64)
        yr = np.zeros((64, k))
        for t, (r, c) in enumerate(sub):
            if r == R:
                yr += tiles[t] @ X1h[c * 64:(c + 1) * 64]
            if c == R and r != R:
                yr += tiles[t].T @ X1h[r * 64:(r + 1) * 64]
        got = Y1[R * 64:(R + 1) * 64].cpu().numpy()
        assert np.abs(got - yr).max() <= 1e-5 * max(1.0, np.abs(yr).max())


@pytest.mark.parametrize("dtype,k,layout", [(torch.float32, 8, "frag"), (torch.float32, 4, "frag"), (torch.float64, 8, "frag"),
                                             (torch.float32, 32, "frag"), (torch.float64, 16, "frag"),
                                             (torch.float32, 16, "tc"), (torch.float64, 8, "tc"),
                                             (torch.float32, 64, "tc"), (torch.float64, 32, "tc"),
                                             (torch.float64, 64, "frag"), (torch.float64, 64, "tc")])
def test_host_batch_pipeline_matches_oracle(pkg, c1_small, dtype, k, layout):
    """cim_sym_spmm_host_batch: host (pinned and pageable, numpy and torch)
    blocks in, host blocks out; every block checked against the oracle, and
    against the single-call operator bit for bit (same kernel, same order)."""
    n, rc, tiles = c1_small
    H = pkg.HalfTiles.synthetic(n, tile_rc=rc, dtype=dtype, layout=layout)
    g = torch.Generator().manual_seed(5)
    Xs = [torch.randn((n, k), generator=g, dtype=dtype).pin_memory() for _ in range(3)]
    Xs.append(torch.randn((n, k), generator=g, dtype=dtype))  # pageable
    Xs.append(Xs[0].numpy().copy())  # numpy
    Ys = pkg.sym_spmm_host_batch(H, Xs)
    assert isinstance(Ys[-1], np.ndarray) and Ys[0].is_pinned()
    tl = tiles if dtype == torch.float32 else tiles.astype(np.float64)
    for X, Y in zip(Xs, Ys):
        Xn = X if isinstance(X, np.ndarray) else X.numpy()
        Yn = Y if isinstance(Y, np.ndarray) else Y.numpy()
        check_result(n, rc, tl, Xn, Yn, dtype)
        Y1 = pkg.sym_spmm(H, torch.from_numpy(Xn).cuda()).cpu().numpy()
        # atomics make the summation order of Y_C run-dependent: compare to the gate, not bits
        assert np.abs(Y1 - Yn).max() <= 1e-5 * np.abs(Y1).max()
    # caller-owned outputs, and validation before any compute
    outs = [torch.empty((n, k), dtype=dtype) for _ in range(2)]
    assert pkg.sym_spmm_host_batch(H, Xs[:2], out=outs) is not None
    with pytest.raises(ValueError):
        pkg.sym_spmm_host_batch(H, [torch.zeros((n + 1, k), dtype=dtype)])
    with pytest.raises(ValueError):
        pkg.sym_spmm_host_batch(H, [torch.zeros((n, k), dtype=dtype, device="cuda")])
    with pytest.raises(ValueError):
        pkg.sym_spmm_host_batch(H, Xs[:2], out=outs[:1])


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("rows,ca,cb", [(1, 1, 1), (1000, 8, 8), (100_003, 24, 48), (70_000, 5, 13), (4096, 64, 64)])
def test_gram_f64_matches_numpy(pkg, dtype, rows, ca, cb):
    """cim_gram: Aᵀ·B with f64 accumulation (LOBPCG's Gram products),
    including strided column views and ragged column counts; reproducible."""
    from paper_2110_10765_b200.lobpcg import gram_f64

    g = torch.Generator().manual_seed(rows + ca)
    base = torch.randn((rows, ca + cb + 3), generator=g, dtype=dtype)
    A, B = base[:, :ca], base[:, 3:3 + cb]  # strided views (lda = ldb = ca+cb+3)
    want = A.double().numpy().T @ B.double().numpy()
    got = gram_f64(A.cuda(), B.cuda()).cpu().numpy()
    tol = 1e-12 * np.sqrt(rows) * (np.abs(A.double().numpy()).T @ np.abs(B.double().numpy())).max()
    assert np.abs(got - want).max() <= tol + 1e-300
    again = gram_f64(A.cuda(), B.cuda()).cpu().numpy()
    assert np.array_equal(got, again)  # fixed reduction order
    with pytest.raises(ValueError):
        gram_f64(A.cuda(), B[:-1].cuda())


@pytest.mark.parametrize("rows,nslots_a,nslots_b,mask", [(100_003, 1, 1, 0), (257, 2, 1, 0), (1_000_000, 3, 6, 0),
                                                         (300_001, 3, 6, 0b000111_000111_000111)])
def test_gram_fast_mode(pkg, rows, nslots_a, nslots_b, mask):
    """cim_gram_blocked_ex with CIM_GRAM_FAST (the eigensolver's f32 Gram):
    f32 products and ≤ 32-row f32 partial sums, f64 across runs — within
    2⁻¹⁸·(|A|ᵀ|B|) of the f64 product, reproducible, masked blocks zero; the
    exact mode on the same block-major operands stays at f64 accuracy."""
    from paper_2110_10765_b200._lib import CIM_F32, CIM_GRAM_FAST, lib

    g = torch.Generator().manual_seed(rows)
    buf = torch.randn((6, rows, 8), generator=g).cuda()
    L = lib()
    ca, cb = 8 * nslots_a, 8 * nslots_b
    need = int(L.cim_gram_workspace_bytes(rows, ca, cb))
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")

    def run(flags):
        out = torch.empty((ca, cb), dtype=torch.float64, device="cuda")
        assert L.cim_gram_blocked_ex(buf[0].data_ptr(), 8, 8, rows * 8, ca, buf[0].data_ptr(), 8, 8, rows * 8, cb,
                                     rows, CIM_F32, out.data_ptr(), ws.data_ptr(), need, mask, flags, None) == 0
        return out.cpu().numpy()

    dense = buf.cpu().double().permute(1, 0, 2).reshape(rows, 48).numpy()
    A, B = dense[:, :ca], dense[:, :cb]
    want = A.T @ B
    absprod = np.abs(A).T @ np.abs(B)
    if mask:
        keep = np.zeros((ca // 8, cb // 8), bool)
        for bi in range(ca // 8):
            for bj in range(cb // 8):
                keep[bi, bj] = (mask >> (bi * (cb // 8) + bj)) & 1
        want = want * np.kron(keep, np.ones((8, 8)))
    fast = run(CIM_GRAM_FAST)
    assert np.abs(fast - want).max() <= 2.0 ** -18 * absprod.max()
    assert np.array_equal(fast, run(CIM_GRAM_FAST))
    exact = run(0)
    assert np.abs(exact - want).max() <= 1e-12 * np.sqrt(rows) * absprod.max()
    assert L.cim_gram_blocked_ex(buf[0].data_ptr(), 8, 8, rows * 8, ca, buf[0].data_ptr(), 8, 8, rows * 8, cb, rows,
                                 CIM_F32, ws.data_ptr(), ws.data_ptr(), need, 0, 4, None) == 1  # unknown flag


@pytest.mark.parametrize("rows,qs,ps", [(1, 1, 1), (100_001, 3, 2), (4099, 2, 1), (70_000, 4, 4), (50_000, 2, 2)])
def test_tsmm_host_c_and_residual(pkg, rows, qs, ps):
    """cim_tsmm_blocked_hc (C from host memory, in the kernel parameters)
    matches cim_tsmm_blocked on block-major slots, including in place
    (p ≤ 16); cim_block_residual = AX − X·diag(λ) with zero padding columns."""
    from paper_2110_10765_b200._lib import lib

    L = lib()
    g = torch.Generator().manual_seed(rows + qs)
    bw = 8
    buf = torch.randn((8, rows, bw), generator=g).cuda()
    q, p = qs * bw, ps * bw
    C = torch.randn((q, p), generator=g)
    out_dev = torch.randn((ps, rows, bw), generator=g).cuda()
    out_hc = out_dev.clone()
    bs = rows * bw
    Cd = C.cuda()
    Ch = C.numpy().astype(np.float32)
    assert L.cim_tsmm_blocked(buf.data_ptr(), bw, bw, bs, q, Cd.data_ptr(), p, -1.0, 1.0, out_dev.data_ptr(), bw, bw,
                              bs, rows, None) == 0
    assert L.cim_tsmm_blocked_hc(buf.data_ptr(), bw, bw, bs, q, Ch.ctypes.data, p, -1.0, 1.0, out_hc.data_ptr(), bw,
                                 bw, bs, rows, None) == 0
    assert torch.equal(out_dev, out_hc)
    if qs == ps and p <= 16:  # in place (one 16-column strip per thread): Out = A·C over the same slots
        want = (buf[:qs].permute(1, 0, 2).reshape(rows, q).double().cpu() @ C.double()).float()
        assert L.cim_tsmm_blocked_hc(buf.data_ptr(), bw, bw, bs, q, Ch.ctypes.data, p, 1.0, 0.0, buf.data_ptr(), bw,
                                     bw, bs, rows, None) == 0
        got = buf[:ps].permute(1, 0, 2).reshape(rows, p).cpu()
        assert (got - want).abs().max().item() <= 1e-4 * want.abs().max().item()
    big = np.zeros((64, 64), np.float32)
    assert L.cim_tsmm_blocked_hc(buf.data_ptr(), bw, bw, bs, 64, big.ctypes.data, 64, 1.0, 0.0, out_hc.data_ptr(), bw,
                                 bw, bs, rows, None) == 3  # > 1024 values: unsupported
    # residual
    m = 5
    lam = np.linspace(-2.0, 3.0, m)
    X = torch.randn((rows, bw), generator=g)
    AX = torch.randn((rows, bw), generator=g)
    X[:, m:] = 0
    AX[:, m:] = 0
    W = torch.full((rows, bw), 7.0).cuda()
    assert L.cim_block_residual(X.cuda().data_ptr(), AX.cuda().data_ptr(), lam.ctypes.data, m, W.data_ptr(), rows, bw,
                                None) == 0
    lam32 = torch.zeros(bw)
    lam32[:m] = torch.from_numpy(lam).float()
    want = AX - X * lam32
    assert (W.cpu() - want).abs().max().item() <= 1e-6 * (want.abs().max().item() + 1)
    assert torch.all(W[:, m:] == 0)


@pytest.mark.parametrize("rows,q,m", [(1, 8, 8), (100_001, 24, 8), (4099, 16, 5), (70_000, 48, 3), (3, 32, 0)])
def test_ritz_update_fused(pkg, rows, q, m):
    """cim_ritz_update_b8 (the LOBPCG Ritz update fused with the next
    residual) = two tsmm over S and AS plus W = AX − X·diag(λ), f64 reference;
    padding columns (C columns ≥ m in each half are zero, λ_j = 0) stay zero."""
    from paper_2110_10765_b200._lib import lib

    L = lib()
    g = torch.Generator().manual_seed(rows + q + m)
    bw, qs = 8, q // 8
    inp = torch.randn((2 * qs, rows, bw), generator=g)  # S slots then AS slots
    C = torch.randn((q, 16), generator=g)
    C[:, m:8] = 0
    C[:, 8 + m:] = 0
    lam = np.linspace(-2.0, 3.0, m)
    out = torch.full((5, rows, bw), 7.0).cuda()
    d = inp.cuda()
    Ch = C.numpy().astype(np.float32)
    bs = rows * bw
    assert L.cim_ritz_update_b8(d[0].data_ptr(), d[qs].data_ptr(), bs, q, Ch.ctypes.data, lam.ctypes.data, m,
                                out.data_ptr(), bs, rows, None) == 0
    S = inp[:qs].permute(1, 0, 2).reshape(rows, q).double()
    AS = inp[qs:].permute(1, 0, 2).reshape(rows, q).double()
    PX, APX = S @ C.double(), AS @ C.double()
    lam_p = torch.zeros(bw, dtype=torch.float64)
    lam_p[:m] = torch.from_numpy(lam)
    want = [PX[:, :8], PX[:, 8:], APX[:, 8:] - PX[:, 8:] * lam_p, APX[:, :8], APX[:, 8:]]
    got = out.cpu().double()
    scale = max(PX.abs().max().item(), APX.abs().max().item(), 1.0) * q
    for s in range(5):
        assert (got[s] - want[s]).abs().max().item() <= 2e-6 * scale, s
        assert torch.all(got[s][:, m:] == 0), s
    assert L.cim_ritz_update_b8(d[0].data_ptr(), d[qs].data_ptr(), bs, 40, Ch.ctypes.data, lam.ctypes.data, m,
                                out.data_ptr(), bs, rows, None) == 1  # q not supported


@pytest.mark.parametrize("rows,q,p,off", [(1, 1, 1, 0), (1000, 8, 8, 0), (100_001, 24, 16, 8), (5000, 7, 5, 3),
                                          (4096, 64, 64, 0)])
def test_tsmm_matches_torch(pkg, rows, q, p, off):
    """cim_tsmm: Out = alpha·A·C + beta·Out into column slices of a wider
    buffer (vector path when everything is 16-byte aligned, scalar otherwise)."""
    from paper_2110_10765_b200.lobpcg import tsmm

    g = torch.Generator().manual_seed(rows + q + p)
    buf = torch.randn((rows, off + q + p + 4), generator=g).cuda()
    A = buf[:, off:off + q]
    Out = buf[:, off + q:off + q + p]
    C = torch.randn((q, p), generator=g, dtype=torch.float64)
    want = (-0.5 * (A.double().cpu() @ C) + 2.0 * Out.double().cpu()).numpy()
    untouched = buf[:, :off].clone()
    tsmm(A, C, Out, alpha=-0.5, beta=2.0)
    got = Out.double().cpu().numpy()
    scale = (np.abs(A.double().cpu().numpy()) @ np.abs(C.numpy())).max() + 1.0
    assert np.abs(got - want).max() <= 4e-6 * scale * q
    assert torch.equal(buf[:, :off], untouched)
    tsmm(A, C, Out)  # beta = 0: Out not read
    assert np.abs(Out.double().cpu().numpy() - (A.double().cpu() @ C).numpy()).max() <= 4e-6 * scale * q


@pytest.mark.parametrize("bands", [2, 3, 7])
def test_column_banded_storage(pkg, c1_small, bands):
    """Tiles stored in column-band order (C // band_cols, R, C): units never
    cross a band, same operator (oracle gates), same tiles after a pack/unpack
    round trip through the permutation."""
    n, rc, tiles = c1_small
    H = pkg.HalfTiles.synthetic(n, tile_rc=rc, bands=bands, max_unit=5)
    assert H.meta["bands"] == bands
    bc = H.meta["band_cols"]
    srt = H.tile_rc_host
    key = (srt[:, 1] // bc).astype(np.int64) * (1 << 40) + srt[:, 0].astype(np.int64) * (1 << 20) + srt[:, 1]
    assert np.all(np.diff(key) > 0)
    assert sorted(map(tuple, srt)) == sorted(map(tuple, rc))
    for u in H.units_host:
        t = srt[u[1]:u[2]]
        assert np.all(t[:, 0] == u[0]) and np.unique(t[:, 1] // bc).size == 1
    for k in (4, 8, 16):
        X = torch.randn((n, k), generator=torch.Generator().manual_seed(k))
        check_result(n, rc, tiles, X.numpy(), pkg.sym_spmm(H, X.cuda()).cpu().numpy(), torch.float32)
    H2 = pkg.HalfTiles.from_dense_tiles(n, rc, tiles, bands=bands)
    back = H2.dense_tiles().cpu().numpy()
    pos = {tuple(r): s for s, r in enumerate(H2.tile_rc_host)}
    for t_in, r in enumerate(rc[:50]):
        assert np.array_equal(back[pos[tuple(r)]], tiles[t_in])



@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("fill", [0.0, 0.02, 0.05, 0.3, 0.9])  # 0.05: every staged tile fits 512-entry stages
@pytest.mark.parametrize("k", [1, 2, 3, 4, 8, 12, 16, 24, 32, 64])
def test_sparse_tiles_vs_oracle(pkg, dtype, fill, k):
    """COO-in-tile storage: random symmetric matrices whose 64-tiles have a
    given fill (ragged n, empty rows, diagonal and off-diagonal tiles), stored
    with the break-even split (fill 0.9 → dense) and forced all-sparse; the
    operator must match the oracle and the all-dense storage."""
    rng = np.random.default_rng(int(fill * 100) + k)
    n = 700
    nb = (n + 63) // 64
    rc = pkg.synthetic_pattern(nb, 0.4, seed=2)
    ii, jj = [], []
    for R, C in rc:
        m = rng.random((64, 64)) < max(fill, 0.002)
        if R == C:
            m = m | m.T
        a, b = np.nonzero(m)
        ii.append(R * 64 + a)
        jj.append(C * 64 + b)
    i = np.concatenate(ii)
    j = np.concatenate(jj)
    ok = (i < n) & (j < n)
    i, j = i[ok], j[ok]
    key = np.unique(np.minimum(i, j) * n + np.maximum(i, j))
    lo, hi = key // n, key % n
    vals = rng.standard_normal(key.size)
    I = np.concatenate([lo, hi[lo != hi]])
    J = np.concatenate([hi, lo[lo != hi]])
    V = np.concatenate([vals, vals[lo != hi]])
    npd = np.float32 if dtype == torch.float32 else np.float64
    V = V.astype(npd)
    X = torch.randn((n, k), generator=torch.Generator().manual_seed(k), dtype=dtype)
    from paper_2110_10765_b200.halftiles import dense_break_even
    H_mix = pkg.HalfTiles.from_coo(n, I, J, V, dtype=dtype, dense_fill=dense_break_even(dtype))
    H_sp = pkg.HalfTiles.from_coo(n, I, J, V, dtype=dtype, dense_fill=2.0)
    H_dn = pkg.HalfTiles.from_coo(n, I, J, V, dtype=dtype, dense_fill=0.0)
    assert H_sp.n_tiles == 0 and H_dn.n_sparse_tiles == 0
    if fill < 0.5:
        assert H_mix.n_sparse_tiles > 0
    if fill == 0.05:  # the forced-sparse storage runs the staged kernel with 512-entry stages
        staged, _ = H_sp.sparse.work_split()
        assert staged.numel() > 0 and H_sp.sparse.descriptor().staged_max_entries <= 512
    rc_all, tiles = H_dn.export_dense()
    for H in (H_mix, H_sp, H_dn):
        Y = pkg.sym_spmm(H, X.cuda()).cpu().numpy()
        check_result(n, rc_all, tiles.astype(np.float64), X.numpy(), Y, dtype)
    # accumulate path and host batch on the mixed storage
    out = torch.ones((n, k), dtype=dtype, device="cuda")
    pkg.sym_spmm(H_mix, X.cuda(), out=out, accumulate=True)
    Y1 = pkg.sym_spmm(H_mix, X.cuda())
    assert (out - 1.0 - Y1).abs().max().item() <= 1e-5 * Y1.abs().max().item() + 1e-6
    if k in (4, 8):
        Yb = pkg.sym_spmm_host_batch(H_mix, [X.pin_memory()])[0]
        assert (Yb.cuda() - Y1).abs().max().item() <= 1e-5 * Y1.abs().max().item() + 1e-6
    # CIM_DETERMINISTIC over sparse tiles: rows / columns walked in stored
    # (ascending) order, so every storage split gives the same bits as the
    # all-dense walk (a zero tile element adds +0 exactly)
    Yd = [pkg.sym_spmm(H, X.cuda(), deterministic=True) for H in (H_dn, H_mix, H_sp)]
    check_result(n, rc_all, tiles.astype(np.float64), X.numpy(), Yd[1].cpu().numpy(), dtype)
    assert torch.equal(Yd[0], Yd[1]) and torch.equal(Yd[0], Yd[2])
    assert torch.equal(Yd[2], pkg.sym_spmm(H_sp, X.cuda(), deterministic=True))


@pytest.mark.parametrize("fill", [0.05, 0.17, 0.6])
def test_synthetic_sparse_device_construction(pkg, fill):
    """Device count → scan → fill (cim_sparse_count_rows / _fill_entries):
    the entry set and values equal the host twin bit for bit, and the
    operator matches the oracle."""
    n = 3000 - 17
    rc = pkg.synthetic_pattern((n + 63) // 64, 0.2, seed=5)
    H = pkg.HalfTiles.synthetic_sparse(n, tile_rc=rc, fill=fill, fill_seed=9, value_seed=3)
    assert H.n_tiles == 0 and H.n_sparse_tiles == rc.shape[0]
    want = oracle.synthetic_sparse_tiles(n, rc, fill, 9, 3)
    got_rc, got = H.export_dense()
    assert np.array_equal(got_rc, rc)
    assert np.array_equal(f32bits(got), f32bits(want))
    assert H.sparse.n_real_entries == int(np.count_nonzero(want))  # h(i^j) is never exactly 0 here
    # the device-built column index equals the host construction from the same entries
    from paper_2110_10765_b200.halftiles import SparseTiles
    tid, r, c, v, _ = H.sparse.to_entries()
    ref = SparseTiles.from_entries(H.sparse.tile_rc_host, tid, r, c, v, torch.float32, "cuda")
    for name in ("rowptr", "colptr", "col", "row", "cperm"):
        assert torch.equal(getattr(H.sparse, name), getattr(ref, name)), name
    X = torch.randn((n, 8), generator=torch.Generator().manual_seed(1))
    check_result(n, rc, want.astype(np.float64), X.numpy(), pkg.sym_spmm(H, X.cuda()).cpu().numpy(), torch.float32)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("k", [1, 4, 8, 16, 32, 64])
@pytest.mark.parametrize("layout", ["frag", "tc"])
def test_deterministic_mode_bitwise_reproducible(pkg, c1_small, dtype, k, layout):
    """CIM_DETERMINISTIC: no float atomics — repeated applies are bitwise
    identical (the atomic path is not, in general), and the result passes the
    oracle gates; accumulate adds onto Y.  Both tile layouts walk the same
    elements in the same order: the same bits."""
    n, rc, tiles = c1_small
    H = pkg.HalfTiles.synthetic(n, tile_rc=rc, dtype=dtype, max_unit=3, layout=layout)
    X = torch.randn((n, k), generator=torch.Generator().manual_seed(k), dtype=dtype).cuda()
    Y1 = pkg.sym_spmm(H, X, deterministic=True)
    Y2 = pkg.sym_spmm(H, X, deterministic=True)
    assert torch.equal(Y1, Y2)
    tl = tiles if dtype == torch.float32 else tiles.astype(np.float64)
    check_result(n, rc, tl, X.cpu().numpy(), Y1.cpu().numpy(), dtype)
    out = torch.ones_like(X)
    pkg.sym_spmm(H, X, out=out, accumulate=True, deterministic=True)
    assert torch.equal(out, Y1 + 1.0)
    if layout == "tc":
        Hf = pkg.HalfTiles.synthetic(n, tile_rc=rc, dtype=dtype, max_unit=3, layout="frag")
        assert torch.equal(Y1, pkg.sym_spmm(Hf, X, deterministic=True))


@pytest.mark.parametrize("name", ["skel_small.npz", "skel_n1024.npz", "skel_identity.npz"])
@pytest.mark.parametrize("dense_fill", [None, 0.0, 2.0])
def test_from_basis_matches_reference_build(pkg, name, dense_fill):
    """GPU construction from the grouped basis (count → scan → fill on the
    device) reproduces the reference build_skeleton's entry set — pair-set
    digest — and value bits, with any dense/sparse split."""
    f = load_fixture(name)
    n = int(f["n"])
    H = pkg.HalfTiles.from_basis(f["basis_occ"], f["basis_bits_lo"], rank=int(f["rank_threshold"]) // 2,
                                 value_seed=int(f["value_seed"]), dense_fill=dense_fill)
    rc, tiles = H.export_dense()
    i, j, v = oracle.half_tiles_to_coo(n, rc, tiles)
    assert oracle.pair_set_digest(i, j) == str(f["pair_digest"])
    got = dict(zip(zip(i.tolist(), j.tolist()), f32bits(v).tolist()))
    want_i, want_j, want_v = f["i"].astype(np.int64), f["j"].astype(np.int64), f32bits(f["v"])
    assert all(got[(a, b)] == c for a, b, c in zip(want_i.tolist(), want_j.tolist(), want_v.tolist()))
    # and the operator on it matches the reference's matrix product
    X = torch.from_numpy(f["X"]).cuda()
    Y = pkg.sym_spmm(H, X).cpu().numpy()
    rel = np.linalg.norm(Y - f["Y_ref"]) / np.linalg.norm(f["Y_ref"])
    assert rel <= 1e-5
    Yd = pkg.sym_spmm(H, X, deterministic=True)
    assert torch.equal(Yd, pkg.sym_spmm(H, X, deterministic=True))
    assert np.linalg.norm(Yd.cpu().numpy() - f["Y_ref"]) / np.linalg.norm(f["Y_ref"]) <= 1e-5


@pytest.mark.parametrize("name", ["skel_small", "skel_n1024", "skel_identity"])
def test_from_basis_file_matches_reference_build(pkg, name):
    """A reference basis file (save_basis format, sampled order) → grouped →
    built on the device: the reference skeleton's pair set and value bits,
    and the operator matches the reference product."""
    meta = json.loads((GOLDEN / "basis_files.json").read_text())[name]
    f = load_fixture(f"{name}.npz")
    H = pkg.HalfTiles.from_basis_file(GOLDEN / f"basis_{name}.txt", group_bits=meta["group_bits"],
                                      rank=int(f["rank_threshold"]) // 2, value_seed=int(f["value_seed"]))
    n = int(f["n"])
    rc, tiles = H.export_dense()
    i, j, v = oracle.half_tiles_to_coo(n, rc, tiles)
    assert oracle.pair_set_digest(i, j) == str(f["pair_digest"])
    X = torch.from_numpy(f["X"]).cuda()
    Y = pkg.sym_spmm(H, X).cpu().numpy()
    assert np.linalg.norm(Y - f["Y_ref"]) / np.linalg.norm(f["Y_ref"]) <= 1e-5
    assert H.meta["n_orbitals"] == f["orb"].shape[0]


@pytest.mark.parametrize("dtype,k", [(torch.float32, 8), (torch.float32, 16), (torch.float64, 8)])
@pytest.mark.parametrize("world", [1, 3, 8])
def test_chunked_apply_virtual_ranks(pkg, dtype, k, world):
    """cim_sym_spmm_chunked — the fused multi-GPU apply's kernel — on one GPU
    with `world` virtual ranks: each rank's balanced panel of tiles runs
    against X / Y split into per-rank row chunks (separate allocations, as
    peer-mapped chunks would be); the assembled Y must match the oracle."""
    from paper_2110_10765_b200.sharded import row_chunks, shard_tile_range, sym_spmm_chunked

    n = 4096 - 37
    nb = (n + 63) // 64
    rc = pkg.synthetic_pattern(nb, 0.2, seed=7)
    units = pkg.plan_units(rc, nb, max_unit=5)
    per, total = row_chunks(n, world)
    g = torch.Generator().manual_seed(world + k)
    X = torch.randn((total, k), generator=g, dtype=dtype)
    X[n:] = 0
    Xc = [X[c * per:(c + 1) * per].clone().cuda() for c in range(world)]
    Yc = [torch.zeros((per, k), dtype=dtype, device="cuda") for _ in range(world)]
    for r in range(world):
        _, _, t0, t1 = shard_tile_range(units, world, r)
        if t1 > t0:
            H = pkg.HalfTiles.synthetic(n, tile_rc=rc[t0:t1], dtype=dtype, max_unit=5)
            sym_spmm_chunked(H, Xc, Yc, per)
    Y = torch.cat([y.cpu() for y in Yc])[:n].numpy()
    tiles = oracle.synthetic_dense_tiles(n, rc, seed=0)
    check_result(n, rc, tiles if dtype == torch.float32 else tiles.astype(np.float64), X[:n].numpy(), Y, dtype)
    with pytest.raises(ValueError):
        sym_spmm_chunked(H, Xc[:1], Yc[:1], 64)  # chunks must cover the rows


@pytest.mark.parametrize("name", ["skel_small.npz", "skel_n1024.npz", "skel_identity.npz"])
def test_reference_pipeline_pins_on_device_storage(pkg, name):
    """The reference's own pipeline pins re-run on the
    device-built storage: conservation — stored pairs = count_pairs total
    (test_pipeline.py:140-145, test_acceptance.py:288-304); the diagonal holds
    h(i,i) = h(0,0,seed) (test_pipeline.py:175-190); and the forward and
    transposed walks agree, ⟨X₁, A X₂⟩ = ⟨A X₁, X₂⟩ (test_pipeline.py:278-286)."""
    f = load_fixture(name)
    n = int(f["n"])
    for H in (pkg.HalfTiles.from_basis(f["basis_occ"], f["basis_bits_lo"], value_seed=int(f["value_seed"])),
              pkg.HalfTiles.from_coo(n, f["i"], f["j"], f["v"], dense_fill=0.5)):
        rc, tiles = H.export_dense()
        i, j, v = oracle.half_tiles_to_coo(n, rc, tiles)
        assert i.size == int(f["whole_pairs"]) == int(f["nnz"])
        d = i == j
        assert np.all(f32bits(v[d]) == int(f["diag_value_bits"]))
        g = torch.Generator().manual_seed(3)
        X1 = torch.randn((n, 8), generator=g, dtype=torch.float64)
        X2 = torch.randn((n, 8), generator=g, dtype=torch.float64)
        H64 = pkg.HalfTiles.from_coo(n, i, j, v.astype(np.float64), dtype=torch.float64)
        A1 = pkg.sym_spmm(H64, X1.cuda()).cpu()
        A2 = pkg.sym_spmm(H64, X2.cuda()).cpu()
        lhs, rhs = (X1 * A2).sum(0), (A1 * X2).sum(0)
        assert torch.allclose(lhs, rhs, rtol=1e-12, atol=1e-12 * float(lhs.abs().max()))


@pytest.mark.parametrize("dtype,k", [(torch.float32, 16), (torch.float32, 8), (torch.float64, 8), (torch.float64, 16)])
def test_tensor_core_kernels_strided_y_and_accumulate(pkg, c1_small, dtype, k):
    """Through the C-ABI: Y a column slice of a wider buffer (ldy = 2k, so the
    bulk-reduction flush falls back to per-row reductions), the neighbouring
    columns untouched, and CIM_ACCUMULATE adding a second product."""
    from paper_2110_10765_b200._lib import CIM_ACCUMULATE, check, lib

    n, rc, tiles = c1_small
    H = pkg.HalfTiles.synthetic(n, tile_rc=rc, dtype=dtype, layout="tc")
    X = torch.randn((H.n_pad, k), generator=torch.Generator().manual_seed(3), dtype=dtype)
    X[n:] = 0
    Xd = X.cuda()
    Yw = torch.full((H.n_pad, 2 * k), 3.0, dtype=dtype, device="cuda")
    Yv = Yw[:, k:]
    s = torch.cuda.current_stream().cuda_stream
    check(lib().cim_sym_spmm(H.descriptor(), Xd.data_ptr(), Yv.data_ptr(), k, k, 2 * k, 0, s), "cim_sym_spmm")
    torch.cuda.synchronize()
    Y1 = Yv.cpu().numpy()[:n]
    check_result(n, rc, tiles.astype(np.float64), X.numpy()[:n], Y1, dtype)
    assert torch.all(Yw[:, :k] == 3.0)
    check(lib().cim_sym_spmm(H.descriptor(), Xd.data_ptr(), Yv.data_ptr(), k, k, 2 * k, CIM_ACCUMULATE, s),
          "cim_sym_spmm")
    torch.cuda.synchronize()
    Y2 = Yv.cpu().numpy()[:n]
    tol = 1e-5 if dtype == torch.float32 else 1e-12
    assert np.abs(Y2 - 2 * Y1).max() <= tol * np.abs(Y1).max()


@pytest.mark.parametrize("dtype,layout,k", [(torch.float32, "frag", 8), (torch.float32, "tc", 16),
                                            (torch.float32, "tc", 40), (torch.float64, "tc", 8),
                                            (torch.float64, "tc", 24), (torch.float64, "frag", 64),
                                            (torch.float32, "frag", 5), (torch.float64, "tc", 3)])
def test_api_layouts_and_accumulate(pkg, c1_small, dtype, layout, k):
    """The public call in its variants on every kernel family: X as (n, k) or
    the reference's (k, n), torch or numpy, `out=` (device / numpy) and
    `accumulate=True`, padded widths — each against the oracle."""
    n, rc, tiles = c1_small
    H = pkg.HalfTiles.synthetic(n, tile_rc=rc, dtype=dtype, layout=layout)
    tl = tiles.astype(np.float64)
    g = torch.Generator().manual_seed(11 + k)
    X = torch.randn((n, k), generator=g, dtype=dtype)
    Y_nk = pkg.sym_spmm(H, X.cuda()).cpu().numpy()
    check_result(n, rc, tl, X.numpy(), Y_nk, dtype)
    # the reference layout (k, n), numpy in → numpy out
    Y_kn = pkg.sym_spmm(H, np.ascontiguousarray(X.numpy().T))
    assert isinstance(Y_kn, np.ndarray) and Y_kn.shape == (k, n)
    tol = 1e-5 if dtype == torch.float32 else 1e-12
    scale = max(1.0, np.abs(Y_nk).max())
    assert np.abs(Y_kn.T - Y_nk).max() <= tol * scale
    # out= on the device, then accumulate into it
    out = torch.empty((n, k), dtype=dtype, device="cuda")
    assert pkg.sym_spmm(H, X.cuda(), out=out) is out
    assert np.abs(out.cpu().numpy() - Y_nk).max() <= tol * scale
    pkg.sym_spmm(H, X.cuda(), out=out, accumulate=True)
    assert np.abs(out.cpu().numpy() - 2 * Y_nk).max() <= 2 * tol * scale
    # out= numpy
    out_np = np.zeros((n, k), dtype=np.float32 if dtype == torch.float32 else np.float64)
    pkg.sym_spmm(H, X.numpy(), out=out_np)
    assert np.abs(out_np - Y_nk).max() <= tol * scale


@pytest.mark.parametrize("dtype,k,layout,kk", [(torch.float32, 3, "frag", 4), (torch.float64, 48, "tc", 64),
                                               (torch.float32, 20, "tc", 24)])
def test_host_batch_rejects_uncompiled_widths(pkg, c1_small, dtype, k, layout, kk):
    """The host-buffer pipeline hands blocks straight to the C-ABI: a width
    without a compiled kernel (which sym_spmm pads or splits into column
    passes on the device) is refused before any copy, naming the width to pad
    to."""
    n, rc, _ = c1_small
    H = pkg.HalfTiles.synthetic(n, tile_rc=rc, dtype=dtype, layout=layout)
    with pytest.raises(ValueError, match=f"pad X to k={kk}"):
        pkg.sym_spmm_host_batch(H, [torch.zeros((n, k), dtype=dtype)])


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_tensor_core_layout_around_the_operator(pkg, tmp_path, dtype):
    """The tensor-core tile layout through the rest of the API: npz save/load
    (values round-trip bit-exactly into the same layout), a reference basis
    built on the device straight into tc tiles (vs the reference's scipy
    product), the fused contraction over a tc pattern (vs the frag pattern),
    and LOBPCG on tc tiles (vs the frag tiles' Ritz values)."""
    from paper_2110_10765_b200.lobpcg import lobpcg_sym

    tol = 1e-5 if dtype == torch.float32 else 1e-12
    f = load_fixture("skel_n1024.npz")
    Hb = pkg.HalfTiles.from_basis(f["basis_occ"], f["basis_bits_lo"], rank=int(f["rank_threshold"]) // 2,
                                  dtype=dtype, layout="tc")
    assert Hb.layout == "tc"
    k = 16
    X = torch.from_numpy(np.ascontiguousarray(np.tile(f["X"], (1, k // f["X"].shape[1] + 1))[:, :k])).to(dtype)
    Yb = pkg.sym_spmm(Hb, X.cuda()).cpu().numpy()
    Hf = pkg.HalfTiles.from_basis(f["basis_occ"], f["basis_bits_lo"], rank=int(f["rank_threshold"]) // 2,
                                  dtype=dtype, layout="frag")
    Yf = pkg.sym_spmm(Hf, X.cuda()).cpu().numpy()
    assert np.abs(Yb - Yf).max() <= tol * max(1.0, np.abs(Yf).max())
    kx = f["X"].shape[1]
    rel = np.linalg.norm(Yb[:, :kx] - f["Y_ref"]) / np.linalg.norm(f["Y_ref"])
    assert rel <= tol
    # save / load keeps the layout and the values
    Hb.save(tmp_path / "tc.npz")
    H2 = pkg.HalfTiles.load(tmp_path / "tc.npz")
    assert H2.layout == "tc" and torch.equal(H2.vals, Hb.vals) and H2.n_sparse_tiles == Hb.n_sparse_tiles
    Y2 = pkg.sym_spmm(H2, X.cuda()).cpu().numpy()
    assert np.abs(Y2 - Yb).max() <= tol * max(1.0, np.abs(Yb).max())
    # LOBPCG on tc tiles: the same lowest Ritz values as on frag tiles
    n = 2048
    rc = pkg.synthetic_pattern(n // 64, 0.1, seed=2)
    Ht = pkg.HalfTiles.synthetic(n, tile_rc=rc, dtype=dtype, layout="tc")
    Hq = pkg.HalfTiles.synthetic(n, tile_rc=rc, dtype=dtype, layout="frag")
    lt = np.sort(lobpcg_sym(Ht, 8, tol=1e-6, max_iter=800, dtype=torch.float64).eigenvalues)
    lq = np.sort(lobpcg_sym(Hq, 8, tol=1e-6, max_iter=800, dtype=torch.float64).eigenvalues)
    assert np.abs(lt - lq).max() <= 1e-4 * np.abs(lq).max()


@pytest.mark.parametrize("layout", ["frag", "tc"])
def test_c_abi_rejects_bad_arguments(pkg, c1_small, layout):
    """cim_sym_spmm validates before any launch: every malformed call returns
    its documented code (EINVAL 1 / EUNSUPPORTED 3) with a message, nothing
    is written to Y, and a good call afterwards still works."""
    import ctypes

    from paper_2110_10765_b200._lib import CIM_EINVAL, CIM_EUNSUPPORTED, lib

    L = lib()
    n, rc, tiles = c1_small
    H = pkg.HalfTiles.synthetic(n, tile_rc=rc, layout=layout)
    d = H.descriptor()
    k = 16
    X = torch.randn((H.n_pad, k), device="cuda")
    Y = torch.full((H.n_pad + 8, k), 7.0, device="cuda")
    st = None
    kb = 12  # no f32 kernel for k = 12 in either layout (16-byte rows, so validation passes)
    cases = [
        (L.cim_sym_spmm(None, X.data_ptr(), Y.data_ptr(), k, k, k, 0, st), CIM_EINVAL),
        (L.cim_sym_spmm(d, 0, Y.data_ptr(), k, k, k, 0, st), CIM_EINVAL),
        (L.cim_sym_spmm(d, X.data_ptr(), 0, k, k, k, 0, st), CIM_EINVAL),
        (L.cim_sym_spmm(d, X.data_ptr() + 4, Y.data_ptr(), k, k, k, 0, st), CIM_EINVAL),  # misaligned X
        (L.cim_sym_spmm(d, X.data_ptr(), Y.data_ptr() + 4, k, k, k, 0, st), CIM_EINVAL),  # misaligned Y
        (L.cim_sym_spmm(d, X.data_ptr(), Y.data_ptr(), k, k, k - 1, 0, st), CIM_EINVAL),  # ldy < k
        (L.cim_sym_spmm(d, X.data_ptr(), Y.data_ptr(), 0, k, k, 0, st), None),
        (L.cim_sym_spmm(d, X.data_ptr(), Y.data_ptr(), 65, 65, 65, 0, st), None),
        (L.cim_sym_spmm(d, X.data_ptr(), Y.data_ptr(), kb, kb, kb, 0, st), CIM_EUNSUPPORTED),  # no kernel
    ]
    for got, want in cases:
        assert got != 0
        if want is not None:
            assert got == want, (got, want)
        assert L.cim_last_error() and len(L.cim_last_error()) > 0
    torch.cuda.synchronize()
    assert torch.all(Y == 7.0)  # nothing written by a refused call
    assert L.cim_sym_spmm(d, X.data_ptr(), Y.data_ptr(), k, k, k, 0, st) == 0
    tl = tiles.astype(np.float64)
    check_result(n, rc, tl, X[:n].cpu().numpy(), Y[:n].cpu().numpy(), torch.float32)


def test_from_basis_chunked_count_identical(pkg, monkeypatch):
    """The candidate tiles are counted in chunks (memory-bounded for bases
    whose block-pair bound keeps most pairs): any chunk size gives the same
    tiles, entry order and value bits."""
    from paper_2110_10765_b200 import construct

    f = load_fixture("skel_n1024.npz")
    args = (f["basis_occ"], f["basis_bits_lo"])
    kw = dict(rank=int(f["rank_threshold"]) // 2, value_seed=int(f["value_seed"]))
    H1 = pkg.HalfTiles.from_basis(*args, **kw)
    monkeypatch.setattr(construct, "COUNT_CHUNK_TILES", 7)
    H2 = pkg.HalfTiles.from_basis(*args, **kw)
    assert np.array_equal(H1.tile_rc_host, H2.tile_rc_host) and torch.equal(H1.vals, H2.vals)
    a, b = H1.export_dense(), H2.export_dense()
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1].view(np.uint32), b[1].view(np.uint32))
    assert H1.meta["candidate_tiles"] == H2.meta["candidate_tiles"]


RANDOM_CASES = int(os.environ.get("CIM_RANDOM_CASES", "60"))  # 600 passed once in 12 s (end of round 2)


@pytest.mark.parametrize("case", range(RANDOM_CASES))
def test_randomized_configurations(pkg, case):
    """Seeded random configurations — n, tile density, dense/sparse mix and
    entry fill, dtype, layout, k (incl. padded widths), work-unit size,
    storage split, CSR on/off — each against the f64 oracle."""
    rng = np.random.default_rng(1000 + case)
    dtype = torch.float32 if rng.random() < 0.6 else torch.float64
    layout = "tc" if rng.random() < 0.5 else "frag"
    n = int(rng.integers(1, 1500))
    nb = (n + 63) // 64
    ks = [1, 2, 3, 4, 5, 8, 9, 12, 16, 20, 24, 32, 40, 48, 64]
    k = int(rng.choice(ks))
    p = float(rng.choice([0.0, 0.05, 0.2, 0.6, 1.0]))
    fill = float(rng.choice([0.01, 0.05, 0.2, 0.5]))
    sparse = rng.random() < 0.5
    if sparse:
        H = pkg.HalfTiles.synthetic_sparse(n, p, fill=fill, seed=case, fill_seed=case + 1, dtype=dtype)
        if rng.random() < 0.5:
            H.use_symmetric_csr(rng.random() < 0.5)
        rc, tiles = H.export_dense()
    else:
        rc = pkg.synthetic_pattern(nb, p, seed=case)
        H = pkg.HalfTiles.synthetic(n, tile_rc=rc, dtype=dtype, layout=layout,
                                    max_unit=int(rng.choice([1, 3, 32])))
        tiles = oracle.synthetic_dense_tiles(n, rc, seed=0)
    X = torch.randn((n, k), generator=torch.Generator().manual_seed(case), dtype=dtype)
    Y = pkg.sym_spmm(H, X.cuda(), layout="nk").cpu().numpy()
    check_result(n, rc, np.asarray(tiles, np.float64), X.numpy(), Y, dtype)


@pytest.mark.parametrize("case", range(int(os.environ.get("CIM_BASIS_CASES", "6"))))
def test_from_basis_randomized_vs_bruteforce(pkg, case):
    """Seeded random bases (orbital count, particle number, size, order,
    rank): the device build's pair set equals the brute-force set of the
    reference predicate (oracle.occ_diff ≤ 2·rank over all pairs) and every
    stored value is h(i XOR j; seed) bit for bit."""
    rng = np.random.default_rng(77 + case)
    n_sp = int(rng.choice([16, 40, 64, 100, 128]))
    npart = int(rng.integers(1, 6))
    n_want = int(rng.integers(50, 400))
    rank = int(rng.integers(1, 3))
    occ = np.unique(np.sort(np.stack([rng.choice(n_sp, npart, replace=False) + 1 for _ in range(n_want)]), axis=1),
                    axis=0).astype(np.uint16)
    occ = occ[rng.permutation(occ.shape[0])]
    if rng.random() < 0.5:  # grouped-like order by the low bits
        lo0 = np.array([sum(1 << (o - 1) for o in row if o <= 64) for row in occ.tolist()], dtype=np.uint64)
        occ = occ[np.argsort(lo0 & np.uint64(0xFF), kind="stable")]
    n = occ.shape[0]
    lo = np.array([sum(1 << (o - 1) for o in row if o <= 64) for row in occ.tolist()], dtype=np.uint64)
    H = pkg.HalfTiles.from_basis(occ, lo, rank=rank, value_seed=case)
    rc, tiles = H.export_dense()
    i, j, v = oracle.half_tiles_to_coo(n, rc, tiles)
    rows = occ.tolist()
    bi, bj = [], []
    for a in range(n):
        for b in range(a, n):
            if oracle.occ_diff(rows[a], rows[b]) <= 2 * rank:
                bi.append(a)
                bj.append(b)
    bi, bj = np.array(bi), np.array(bj)
    off = bi != bj
    I = np.concatenate([bi, bj[off]])
    J = np.concatenate([bj, bi[off]])
    assert oracle.pair_set_digest(i, j) == oracle.pair_set_digest(I, J)
    want = oracle.h_values(i, j, case)
    assert np.array_equal(np.asarray(v, np.float32).view(np.uint32), np.asarray(want, np.float32).view(np.uint32))


@pytest.mark.parametrize("case", range(int(os.environ.get("CIM_CONTRACT_CASES", "10"))))
def test_contract_pattern_randomized(pkg, case):
    """Seeded random stored patterns (n, tile density, per-tile fill, dense /
    sparse split), vector and operator counts, operator kind, dtype and tile
    layout: the fused contraction matches the f64 oracle within the
    reference's tolerance, forward and transposed."""
    rng = np.random.default_rng(300 + case)
    dtype = torch.float64 if rng.random() < 0.4 else torch.float32
    layout = "tc" if rng.random() < 0.5 else "frag"
    n = int(rng.integers(10, 900))
    nb = (n + 63) // 64
    rc = pkg.synthetic_pattern(nb, float(rng.choice([0.1, 0.4, 1.0])), seed=case)
    ii, jj = [], []
    for R, C in rc:
        m = rng.random((64, 64)) < float(rng.choice([0.02, 0.2, 0.95]))
        if R == C:
            m = m | m.T
        a, b = np.nonzero(m)
        ii.append(R * 64 + a)
        jj.append(C * 64 + b)
    i, j = np.concatenate(ii), np.concatenate(jj)
    ok = (i < n) & (j < n)
    key = np.unique(np.minimum(i[ok], j[ok]) * n + np.maximum(i[ok], j[ok]))
    lo, hi = key // n, key % n
    I = np.concatenate([lo, hi[lo != hi]])
    J = np.concatenate([hi, lo[lo != hi]])
    if I.size == 0:
        I, J = np.array([0]), np.array([0])
    pattern = pkg.HalfTiles.from_coo(n, I, J, np.ones(I.size), dtype=dtype, layout=layout)
    n_vec, m_ops = int(rng.integers(1, 21)), int(rng.integers(1, 20))
    op_kind = "identity" if rng.random() < 0.2 else "symmetric_hash"
    c = pkg.random_coefficients(n_vec, n, seed=case, kind="gauss")
    inp = pkg.ObservablesInput(c=c, m_ops=m_ops, op_kind=op_kind, seed=case + 5)
    got = pkg.contract_pattern(pattern, inp).astype(np.float64)
    want = oracle.contract_vmv(c, I, J, m_ops, {"symmetric_hash": 1, "identity": 0}[op_kind], case + 5)
    tol = oracle.contraction_tolerance(c, I.size)
    assert np.abs(got - want).max() <= tol
    got_t = pkg.contract_pattern(pattern, pkg.ObservablesInput(c=c, m_ops=m_ops, op_kind=op_kind, seed=case + 5),
                                 transpose=True)
    assert np.abs(got_t - got).max() <= tol


def test_square_input_needs_an_explicit_layout(pkg):
    """X of shape (n, n) reads the same as (n, k) and the reference's (k, n):
    "auto" refuses it; an explicit layout applies it either way."""
    n = 40
    H = pkg.HalfTiles.synthetic(n, p=1.0, seed=1)
    X = torch.randn((n, n), generator=torch.Generator().manual_seed(1))
    with pytest.raises(ValueError, match="indistinguishable"):
        pkg.sym_spmm(H, X.cuda())
    Y_nk = pkg.sym_spmm(H, X.cuda(), layout="nk")
    Y_kn = pkg.sym_spmm(H, X.t().contiguous().cuda(), layout="kn")
    assert torch.allclose(Y_nk, Y_kn.t(), rtol=0, atol=1e-5 * Y_nk.abs().max().item())
