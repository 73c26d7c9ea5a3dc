"""Where does rs_score_poses (host buffers) spend its time beyond the kernel?  C3, 10^6 poses:
the device-resident async launch, the synchronous call on device buffers (chunked launches, no
copies) and on pinned host buffers (chunked copies + launches)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import __graft_entry__
__graft_entry__.build_library()
from paper_2510_26611_b200 import rsdock
from synth import configs as syn

w = syn.config_c3()
prot = rsdock.Protein(w.protein_q, w.protein_xyz, w.box_half_width, **w.params())
dev = torch.device("cuda:0")
P, L = w.P, w.L
q, y = torch.tensor(w.ligand_q, device=dev), torch.tensor(w.ligand_xyz, device=dev).contiguous()
ps = torch.tensor(w.poses, device=dev).contiguous()
E = torch.empty(P, dtype=torch.float64, device=dev)
D = torch.empty(P, dtype=torch.float64, device=dev)
hp = torch.from_numpy(w.poses).pin_memory()
hq = torch.from_numpy(w.ligand_q).pin_memory()
hy = torch.from_numpy(np.ascontiguousarray(w.ligand_xyz)).pin_memory()
hE = torch.empty(P, dtype=torch.float64).pin_memory()
hD = torch.empty(P, dtype=torch.float64).pin_memory()


def t(f, k=7):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(k):
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(ts))


cnt = torch.zeros(1, dtype=torch.int64, device=dev)
print("async device launch    %.4f ms" % t(lambda: prot.score_async(q, y, ps, E, D, cnt)))
print("sync, device buffers   %.4f ms" % t(lambda: rsdock.rs_score_poses(prot.handle, q, y, L, ps, P, E, D)))
print("sync, host poses only  %.4f ms" % t(lambda: rsdock.rs_score_poses(prot.handle, q, y, L, hp, P, E, D)))
print("sync, host outs only   %.4f ms" % t(lambda: rsdock.rs_score_poses(prot.handle, q, y, L, ps, P, hE, hD)))
print("sync, all host         %.4f ms" % t(lambda: rsdock.rs_score_poses(prot.handle, hq, hy, L, hp, P, hE, hD)))
