"""CPU-side checks: the C-ABI library loads and exports every symbol the
header declares; the native planner/partitioner; the synthetic pattern; the
host fragment map agrees with the header's formula.  No GPU compute here."""

import re
from pathlib import Path

import numpy as np
import pytest

import paper_2110_10765_b200 as pkg
from paper_2110_10765_b200 import _lib
from paper_2110_10765_b200.halftiles import fragment_pack_host

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "cim_b200.h").read_text()
    return sorted(set(re.findall(r"CIM_API\s+[\w\s\*]*?\b(cim_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = pkg.lib()
    syms = header_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTS)
    assert b"sm_100a" in L.cim_version()


def test_library_is_built_for_sm100a():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_struct_layout_matches_header(tmp_path):
    """Every field of the ctypes mirrors sits where a C compiler puts it in
    include/cim_b200.h (offsets and sizes from gcc on the header itself)."""
    import ctypes
    import shutil
    import subprocess

    structs = {"cim_half_tiles": pkg._lib.CimHalfTiles, "cim_sparse_tiles": pkg._lib.CimSparseTiles}
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "cim_b200.h"', "int main(void) {"]
    for cname, cls in structs.items():
        lines.append(f'printf("{cname} sizeof %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    root = Path(__file__).resolve().parent.parent
    subprocess.run(["gcc", "-std=c11", "-I", str(root / "include"), str(src), "-o", str(exe)], check=True)
    got = {}
    for line in subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.splitlines():
        cname, field, val = line.split()
        got[(cname, field)] = int(val)
    for cname, cls in structs.items():
        assert got[(cname, "sizeof")] == ctypes.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert got[(cname, fname)] == getattr(cls, fname).offset, (cname, fname)


def test_supported_k_table():
    for k in (1, 2, 4, 8, 16, 24, 32, 64):
        assert pkg.supported_k(__import__("torch").float32, k)
    import torch

    assert not pkg.supported_k(torch.float32, 3)
    assert pkg.padded_k(torch.float32, 3) == 4
    assert pkg.padded_k(torch.float32, 5) == 8
    assert pkg.padded_k(torch.float64, 6) == 8
    assert pkg.padded_k(torch.float64, 12) == 12
    assert pkg.padded_k(torch.float64, 20, "tc") == 24
    assert pkg.padded_k(torch.float64, 40, "tc") == 64  # two DMMA column passes of 32
    assert pkg.padded_k(torch.float32, 3, "tc") == 8
    assert pkg.padded_k(torch.float32, 9, "tc") == 16
    assert pkg.padded_k(torch.float32, 24, "tc") == 24
    assert pkg.padded_k(torch.float32, 33, "tc") == 40


class TestPlanUnits:
    def test_units_cover_rows_and_respect_max(self):
        rc = pkg.synthetic_pattern(300, 0.2, seed=1)
        u = pkg.plan_units(rc, 300, max_unit=5)
        assert u[0, 1] == 0 and u[-1, 2] == rc.shape[0]
        assert np.all(u[1:, 1] == u[:-1, 2])
        assert np.all(u[:, 2] - u[:, 1] <= 5) and np.all(u[:, 2] > u[:, 1])
        for R, t0, t1, _ in u:
            assert np.all(rc[t0:t1, 0] == R)

    @pytest.mark.parametrize("bad", [
        [[0, 0], [1, 0]],          # below the diagonal
        [[1, 1], [0, 0]],          # rows unsorted
        [[0, 1], [0, 1]],          # duplicate
        [[0, 0], [0, 9]],          # column out of range
    ])
    def test_rejects_bad_tile_lists(self, bad):
        with pytest.raises(ValueError):
            pkg.plan_units(np.array(bad, np.int32), 4)

    def test_partition_is_balanced_and_row_aligned(self):
        nb = 4096
        rc = pkg.synthetic_pattern(nb, 0.01, seed=0)
        u = pkg.plan_units(rc, nb, max_unit=4)
        for parts in (2, 4, 8):
            b = pkg.partition_units(u, parts)
            assert b[0] == 0 and b[-1] == u.shape[0] and np.all(np.diff(b) >= 0)
            tiles = [int(u[b[q + 1] - 1, 2] - u[b[q], 1]) for q in range(parts)]
            assert max(tiles) - min(tiles) <= 0.05 * sum(tiles) / parts + 64
            for q in range(1, parts):
                if 0 < b[q] < u.shape[0]:
                    assert u[b[q], 0] != u[b[q] - 1, 0]  # rows never straddle ranks


class TestSyntheticPattern:
    def test_c1_tile_count(self):
        # nb=1024, p=0.01, seed 0 → 5,244 off-diagonal tiles
        rc = pkg.synthetic_pattern(1024, 0.01, seed=0)
        assert rc.shape[0] == 1024 + 5244
        assert np.all(rc[:, 0] <= rc[:, 1])

    def test_large_grid_geometric_sampling(self):
        nb = 65536
        p = 422745 / (nb * (nb - 1) // 2)
        rc = pkg.synthetic_pattern(nb, p, seed=0)
        off = rc[rc[:, 0] != rc[:, 1]]
        assert abs(off.shape[0] - 422745) < 5 * np.sqrt(422745)
        assert np.all(off[:, 0] < off[:, 1]) and off[:, 1].max() < nb
        key = rc[:, 0].astype(np.int64) * nb + rc[:, 1]
        assert np.all(np.diff(key) > 0)  # sorted, unique
        assert np.array_equal(rc, pkg.synthetic_pattern(nb, p, seed=0))


def test_tc_map_matches_header_formula():
    from paper_2110_10765_b200.halftiles import tc_index_map

    m = tc_index_map()
    assert np.array_equal(np.sort(m), np.arange(4096))  # a permutation
    for r in (0, 3, 5, 63):
        for c in (0, 7, 31, 32, 63):
            byte = r * 256 + (((c // 4) ^ (r % 8)) * 16) + (c % 4) * 4
            assert m[byte // 4] == r * 64 + c


def test_fragment_map_matches_header_formula():
    t = np.arange(4096, dtype=np.float32).reshape(1, 64, 64)
    f = fragment_pack_host(t)[0]
    # vals[t][i][mb][j] = T[rg + 8i][cg + 16j], rg=(mb&31)>>2, cg=4(mb>>5)+(mb&3)
    for i in (0, 3, 7):
        for mb in (0, 5, 37, 127):
            for j in range(4):
                rg = (mb & 31) >> 2
                cg = 4 * (mb >> 5) + (mb & 3)
                assert f[(i * 128 + mb) * 4 + j] == t[0, rg + 8 * i, cg + 16 * j]
    assert np.array_equal(np.sort(f), np.arange(4096, dtype=np.float32))  # a permutation
    t64 = t.astype(np.float64)
    f64 = fragment_pack_host(t64)[0]
    assert np.array_equal(np.sort(f64), np.arange(4096, dtype=np.float64))


def test_halftiles_requires_cuda_device():
    with pytest.raises(ValueError):
        pkg.HalfTiles.synthetic(128, p=0.5, device="cpu")


def test_bench_writes_reference_csv(tmp_path):
    """bench.py --csv: the reference harness's 8-column CSV (cimotifs
    bench.py:54, emit_csv :335-349) — header, one spmm row, '#' metadata."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench", ROOT / "bench.py")
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    line = {"metric": "m", "unit": "GFLOP/s", "dtype": "f32", "n_gpus": 1, "steps": 7, "ms_per_step": 1.5,
            "value": 39000.0, "config": {"workload": "C2", "n": 4194304, "k": 8},
            "roofline": {"frac": 0.77, "achieved": 5000.0}, "e2e": {"value": 19000.0},
            "clocks": {"sm_mhz": 1965.0, "reasons": []}}
    out = tmp_path / "b.csv"
    bench.write_reference_csv(out, line, "frag-1gpu")
    rows = [r for r in out.read_text().splitlines() if r and not r.startswith("#")]
    assert tuple(rows[0].split(",")) == bench.CSV_COLUMNS == (
        "motif", "variant", "n", "m", "particles", "reps", "seconds", "rate")
    cells = rows[1].split(",")
    assert len(cells) == 8 and cells[0] == "spmm" and cells[2] == "4194304" and cells[3] == "8"
    assert float(cells[6]) == 1.5e-3 and float(cells[7]) == 39000.0 and cells[4] == ""
    assert any(r.startswith("# results-digest=") for r in out.read_text().splitlines())


@pytest.mark.parametrize("name", ["skel_small.npz", "skel_n1024.npz", "skel_identity.npz"])
def test_basis_block_bound_never_drops_an_entry(name):
    """construct.candidate_tiles prunes 64-block pairs with a popcount lower
    bound; every block pair holding a reference entry must survive it."""
    from paper_2110_10765_b200.construct import block_bounds, candidate_tiles

    f = np.load(ROOT / "tests" / "golden" / name)
    a, o = block_bounds(f["basis_bits_lo"])
    cand = candidate_tiles(a, o, int(f["rank_threshold"]))
    R, C = f["i"].astype(np.int64) // 64, f["j"].astype(np.int64) // 64
    keep = R <= C
    need = set(zip(R[keep].tolist(), C[keep].tolist()))
    assert need <= set(map(tuple, cand.tolist()))
    assert np.all(cand[:, 0] <= cand[:, 1])


def test_integration_doc_struct_matches_header():
    """The ctypes stub INTEGRATION.md tells reference maintainers to add lists
    every cim_half_tiles field in order (a short struct would let the library
    read past it)."""
    import re

    doc = (Path(__file__).resolve().parent.parent / "INTEGRATION.md").read_text()
    block = doc[doc.index("class cim_half_tiles(ctypes.Structure):"):]
    block = block[:block.index("\n\n")]  # the class body ends at the first blank line
    names = re.findall(r'\("([a-z_]+)", ctypes\.', block)
    assert names == [f for f, _ in pkg._lib.CimHalfTiles._fields_]


@pytest.mark.parametrize("case", range(12))
def test_plan_and_partition_randomized(case):
    """Seeded random tile lists (size, density, unit cap, part count, incl.
    more parts than block rows): units cover every tile once inside one block
    row and respect the cap; partitions are monotone, cover every unit,
    never split a block row across parts and stay balanced (native planner,
    no GPU)."""
    rng = np.random.default_rng(case)
    nb = int(rng.integers(1, 3000))
    p = float(rng.choice([0.0, 0.001, 0.01, 0.2, 1.0 if nb < 200 else 0.05]))
    rc = pkg.synthetic_pattern(nb, p, seed=case)
    mu = int(rng.choice([1, 2, 7, 32]))
    u = pkg.plan_units(rc, nb, max_unit=mu)
    assert u[0, 1] == 0 and u[-1, 2] == rc.shape[0]
    assert np.all(u[1:, 1] == u[:-1, 2]) and np.all(u[:, 2] - u[:, 1] <= mu) and np.all(u[:, 2] > u[:, 1])
    for R, t0, t1, _ in u[:: max(1, u.shape[0] // 200)]:
        assert np.all(rc[t0:t1, 0] == R)
    parts = int(rng.integers(1, 9))
    b = pkg.partition_units(u, parts)
    assert b[0] == 0 and b[-1] == u.shape[0] and np.all(np.diff(b) >= 0)
    for q in range(1, parts):
        if 0 < b[q] < u.shape[0]:
            assert u[b[q], 0] != u[b[q] - 1, 0]
    tiles = [int(u[b[q + 1] - 1, 2] - u[b[q], 1]) if b[q + 1] > b[q] else 0 for q in range(parts)]
    assert sum(tiles) == rc.shape[0]
    # balance: no part exceeds the ideal share by more than the largest block row (rows are indivisible)
    row_tiles = np.bincount(rc[:, 0], minlength=nb).max()
    assert max(tiles) <= rc.shape[0] / parts + row_tiles + 1
