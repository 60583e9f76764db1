"""Role timers of the tensor-core kernel (CIM_TC_PROFILE=1): one C2 apply."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["CIM_TC_PROFILE"] = "1"
import paper_2110_10765_b200 as pkg

n = 1 << 22
H = pkg.HalfTiles.synthetic(n, n_off=488281 - 65536, seed=0, layout="tc")
X = torch.randn((n, 8), device="cuda")
for _ in range(3):
    Y = pkg.sym_spmm(H, X)
torch.cuda.synchronize()
L = pkg.lib()
buf = np.zeros((1024, 4, 16), np.uint64)
L.cim_tc_profile_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
nct = L.cim_tc_profile_read(buf.ctypes.data, 1024)
b = buf[:nct].astype(np.float64)
names = ["spl_wait_full", "spl_wait_adir", "spl_work", "mma_wait_split", "mma_wait_tr", "mma_wait_dir",
         "mma_wait_meta", "mma_issue", "epi_wait_meta", "epi_wait_tr", "epi_wait_dir", "epi_work", "tiles", "total"]
roles = ["mma", "splitter0", "splitter1", "epilogue"]
for r, role in enumerate(roles):
    tot = b[:, r, 13].mean()
    vals = {names[i]: b[:, r, i].mean() / max(tot, 1) for i in range(12) if b[:, r, i].mean() > 0}
    print(role, f"total={tot:.0f} cyc", "tiles=%.0f" % b[:, r, 12].mean() if r == 0 else "",
          {k: round(v, 3) for k, v in vals.items()})
