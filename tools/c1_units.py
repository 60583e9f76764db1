"""C1 (n = 65,536, p = 0.01, k = 8 f32) kernel time vs work-unit size, L2
flushed before every apply: the small config is latency-bound (≈ 14 tiles
per ring), so finer units spread it over more rings."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_10765_b200 as b2
from paper_2110_10765_b200._lib import CIM_ACCUMULATE, check, lib

n, k = 65536, 8
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
X = torch.randn((n, k), device="cuda")
Y = torch.zeros_like(X)
out = []
for mu in (32, 8, 4, 2, 1):
    H = b2.HalfTiles.synthetic(n, p=0.01, seed=0, max_unit=mu)
    ts = []
    for rep in range(60):
        flush.zero_()
        Y.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        check(lib().cim_sym_spmm(H.descriptor(), X.data_ptr(), Y.data_ptr(), k, k, k, CIM_ACCUMULATE,
                                 torch.cuda.current_stream().cuda_stream), "spmm")
        b.record()
        torch.cuda.synchronize()
        if rep >= 10:
            ts.append(a.elapsed_time(b))
    ts.sort()
    out.append({"max_unit": mu, "units": int(H.units_host.shape[0]), "kernel_us_median": round(1e3 * ts[len(ts) // 2], 2),
                "rings": os.environ.get("CIM_K8_RINGS", "3")})
print(json.dumps(out))
