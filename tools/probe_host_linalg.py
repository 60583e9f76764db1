"""Host cost of the eigensolver's small dense problems (numpy LAPACK), with
the default BLAS thread pool and limited to one thread."""
import time
import numpy as np
from threadpoolctl import threadpool_limits, threadpool_info


def bench(n, reps=2000):
    rng = np.random.default_rng(0)
    A = rng.standard_normal((n, n))
    A = A @ A.T + n * np.eye(n)
    t0 = time.perf_counter()
    for _ in range(reps):
        np.linalg.eigh(A)
    return (time.perf_counter() - t0) / reps * 1e6


print([(d["internal_api"], d["num_threads"]) for d in threadpool_info()])
for n in (8, 24):
    print(f"eigh {n}x{n}: default {bench(n):.1f} us", end="; ")
    with threadpool_limits(1):
        print(f"1 thread {bench(n):.1f} us")
