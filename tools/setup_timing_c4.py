import sys, time; sys.path.insert(0, ".")
from paper_2510_26611_b200 import rsdock
from synth import configs as syn
w = syn.config_c4(n_poses=16)
import torch; torch.cuda.init()
for fl in (rsdock.RS_FLAG_DEVICE_FFT, rsdock.RS_FLAG_DEVICE_FFT):
    t = time.perf_counter()
    p = rsdock.Protein(w.protein_q, w.protein_xyz, w.box_half_width, **w.params(), flags=fl)
    print("flags", fl, "setup_s", p.info["setup_seconds"], "wall", time.perf_counter() - t, "err", p.info["sampled_max_err"], flush=True)
