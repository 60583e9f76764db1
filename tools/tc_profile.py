"""Role timers of the split-TF32 tensor-core kernel (library built with
-DCIM_TC_PROF, e.g. tools/build_variant.sh tc_prof -DCIM_TC_PROF, loaded via
CIM_B200_LIB): one C2 apply at the given k.  Usage: python tools/tc_profile.py [k]"""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_10765_b200 as pkg

k = int(sys.argv[1]) if len(sys.argv) > 1 else 16
n = 1 << 22
H = pkg.HalfTiles.synthetic(n, n_off=488281 - 65536, seed=0, layout="tc")
X = torch.randn((n, k), device="cuda")
for _ in range(3):
    Y = pkg.sym_spmm(H, X)
torch.cuda.synchronize()
L = pkg.lib()
buf = np.zeros((160, 6, 16), np.uint64)
L.cim_tc_profile_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
nct = L.cim_tc_profile_read(buf.ctypes.data, 160)
b = buf[:nct].astype(np.float64)
slots = {0: ["wait_split", "wait_d_empty", "", "issue"],
         1: ["wait_full", "wait_ab_empty", "", "t_split", "build_b+arrive", "wait_st+fence", "loop"],
         2: ["wait_full", "wait_ab_empty", "", "t_split", "build_b+arrive", "wait_st+fence", "loop"],
         3: ["wait_meta", "wait_d_full", "", "work"],
         4: ["wait_meta", "wait_d_full", "", "work"],
         5: ["wait_empty", "", "", "work"]}
roles = ["mma", "splitter rows", "splitter cols", "epilogue direct", "epilogue transposed", "producer"]
for r, role in enumerate(roles):
    tot = b[:, r, 15].mean()
    tiles = b[:, r, 14].mean()
    vals = {slots[r][i]: round(b[:, r, i].mean() / max(tot, 1), 3) for i in range(7)
            if i < len(slots[r]) and slots[r][i] and b[:, r, i].mean() > 0}
    print(f"k={k} {role:20s} total={tot:.0f} cyc tiles={tiles:.0f} cyc/tile={tot / max(tiles, 1):.0f}", vals)
