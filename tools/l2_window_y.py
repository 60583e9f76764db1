"""A/B: an L2 persisting access-policy window over Y (the random side's
read-modify-write target) for the C2 headline apply (f32 k = 8, frag).
Round 1 tried a window over X (no gain); the verdict suggested Y."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from cuda.bindings import runtime as cudart
import paper_2110_10765_b200 as b2
from paper_2110_10765_b200._lib import CIM_ACCUMULATE, check, lib

dev = 0
n, k = 1 << 22, 8
H = b2.HalfTiles.synthetic(n, n_off=488281 - 65536, seed=0)
X = torch.randn((n, k), device="cuda")
Y = torch.zeros_like(X)
st = torch.cuda.current_stream()
_, maxwin = cudart.cudaDeviceGetAttribute(cudart.cudaDeviceAttr.cudaDevAttrMaxAccessPolicyWindowSize, dev)
_, maxpers = cudart.cudaDeviceGetAttribute(cudart.cudaDeviceAttr.cudaDevAttrMaxPersistingL2CacheSize, dev)
print(json.dumps({"max_window_bytes": maxwin, "max_persisting_l2_bytes": maxpers}))


def timeit(reps=20):
    for _ in range(3):
        Y.zero_()
        check(lib().cim_sym_spmm(H.descriptor(), X.data_ptr(), Y.data_ptr(), k, k, k, CIM_ACCUMULATE, st.cuda_stream), "spmm")
    ts = []
    for _ in range(reps):
        Y.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        check(lib().cim_sym_spmm(H.descriptor(), X.data_ptr(), Y.data_ptr(), k, k, k, CIM_ACCUMULATE, st.cuda_stream), "spmm")
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return round(ts[len(ts) // 2], 4)


def set_window(ptr, nbytes, ratio):
    v = cudart.cudaStreamAttrValue()
    v.accessPolicyWindow.base_ptr = ptr
    v.accessPolicyWindow.num_bytes = nbytes
    v.accessPolicyWindow.hitRatio = ratio
    v.accessPolicyWindow.hitProp = cudart.cudaAccessProperty.cudaAccessPropertyPersisting
    v.accessPolicyWindow.missProp = cudart.cudaAccessProperty.cudaAccessPropertyStreaming
    err, = cudart.cudaStreamSetAttribute(st.cuda_stream, cudart.cudaStreamAttrID.cudaLaunchAttributeAccessPolicyWindow, v)
    return int(err)


res = {"none": timeit()}
err, = cudart.cudaDeviceSetLimit(cudart.cudaLimit.cudaLimitPersistingL2CacheSize, maxpers)
ybytes = Y.numel() * 4
for name, ptr, nb, ratio in [("Y_full_ratio", Y.data_ptr(), min(maxwin, ybytes), min(1.0, maxpers / ybytes)),
                             ("Y_half", Y.data_ptr(), min(maxwin, ybytes // 2), 1.0),
                             ("Y_maxwin_r1", Y.data_ptr(), maxwin, 1.0),
                             ("X_full_ratio", X.data_ptr(), min(maxwin, ybytes), min(1.0, maxpers / ybytes))]:
    e = set_window(ptr, int(nb), float(ratio))
    res[name] = {"err": e, "num_bytes": int(nb), "hitRatio": round(float(ratio), 3), "ms": timeit() if e == 0 else None}
    set_window(ptr, 0, 0.0)
    cudart.cudaCtxResetPersistingL2Cache()
res["none_again"] = timeit()
print(json.dumps(res))
