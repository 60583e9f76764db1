"""Micro-benchmark of the eigensolver block kernels (cim_gram, cim_tsmm) at
C5 shapes (n = 2^22 rows, column slices of a 48-column f32 work buffer)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_10765_b200.lobpcg import gram_f64, tsmm

n = 1 << 22
buf = torch.randn((n, 48), device="cuda")


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


for (c0, c1, d0, d1) in [(16, 24, 16, 24), (0, 16, 16, 24), (0, 24, 0, 48), (8, 16, 0, 48)]:
    A, B = buf[:, c0:c1], buf[:, d0:d1]
    us = timeit(lambda: gram_f64(A, B))
    by = n * ((c1 - c0) + (d1 - d0)) * 4
    print(f"gram {c1-c0:2d}x{d1-d0:2d}: {us:8.1f} us  {by/us/1e3:7.1f} GB/s")
for (a0, a1, o0, o1) in [(0, 16, 16, 24), (16, 24, 40, 48), (0, 24, 24, 40)]:
    A, O = buf[:, a0:a1], buf[:, o0:o1]
    C = torch.randn((a1 - a0, o1 - o0), dtype=torch.float64)
    us = timeit(lambda: tsmm(A, C, O, alpha=-1.0, beta=1.0))
    by = n * ((a1 - a0) + 2 * (o1 - o0)) * 4
    print(f"tsmm {a1-a0:2d}->{o1-o0:2d}: {us:8.1f} us  {by/us/1e3:7.1f} GB/s")
Ac = buf[:, :24].contiguous()
C = torch.randn((24, 16), device="cuda")
us = timeit(lambda: Ac @ C)
print(f"torch mm 24->16 (contiguous): {us:8.1f} us")

# block-major work buffer (what lobpcg uses): 6 slots of (n, 8)
import numpy as np
from paper_2110_10765_b200.lobpcg import _Work
w = _Work(n, 8, torch.float32, torch.device("cuda"), fast_gram=True)
w.buf.normal_()
ex = _Work(n, 8, torch.float32, torch.device("cuda"))
ex.buf.copy_(w.buf)
# lobpcg's MG product: [P X W]ᵀ·[P X W AP AX AW], upper slot blocks of SᵀS and SᵀAS
MG_MASK = 0
for bi in range(3):
    for bj in range(bi, 3):
        MG_MASK |= 1 << (bi * 6 + bj)
        MG_MASK |= 1 << (bi * 6 + 3 + bj)
w2 = _Work(n, 8, torch.float32, torch.device("cuda"))
for (a0, a1, b0, b1, mask) in [(2, 3, 2, 3, 0), (0, 2, 2, 3, 0), (0, 3, 0, 6, 0), (0, 3, 0, 6, MG_MASK)]:
    for name, ww in (("fast", w), ("exact", ex)):
        us = timeit(lambda: ww.gram(a0, a1, b0, b1, None, block_mask=mask))
        print(f"blocked gram {name:5s} {8*(a1-a0):2d}x{8*(b1-b0):2d} mask={mask:#x}: {us:8.1f} us  "
              f"{n*8*max(a1, b1)*4/us/1e3:7.1f} GB/s (incl. host sync)")
C = np.random.default_rng(0).standard_normal((24, 16))
us = timeit(lambda: w.tsmm(0, 3, C, w2, 0, 2))
print(f"blocked tsmm 24->16: {us:8.1f} us  {n*40*4/us/1e3:7.1f} GB/s")
