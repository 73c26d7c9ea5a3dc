set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "device_fft or device_core" 2>&1 | tail -15
python - <<'PY'
import time, sys
sys.path.insert(0, ".")
import torch
from synth import configs as syn
from paper_2510_26611_b200 import rsdock
w = syn.config_c4(n_poses=10)
for fl in (0, rsdock.RS_FLAG_DEVICE_FFT):
    t0 = time.time()
    p = rsdock.Protein(w.protein_q, w.protein_xyz, w.box_half_width, **w.params(), flags=fl)
    print("C4 setup flags", fl, round(time.time() - t0, 2), p.info["sampled_max_err"], p.info["cp_core_err"])
PY
