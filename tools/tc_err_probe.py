import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from conftest import load_golden, golden_model
import paper_1702_07482_b200 as tn
from paper_1702_07482_b200 import _lib
name = sys.argv[1] if len(sys.argv) > 1 else "zeros_in_f"
g = load_golden(name)
model = golden_model(g)
for mode in (1, 2):
    _lib.set_stage_kernel(mode)
    u, _ = tn.run_diffusion(g["f"], model)
    ref = g["u"]
    rel = np.abs(u - ref) / np.maximum(np.abs(ref), 1e-30)
    rel[ref < 1e-6] = 0
    idx = np.argsort(rel.ravel())[::-1][:6]
    print("mode", mode, "max rel", rel.max())
    for i in idx:
        y, x = np.unravel_index(i, ref.shape)
        print(f"  ({y},{x}) ref={ref[y,x]:.6g} gpu={u[y,x]:.6g} rel={rel[y,x]:.3g} f={g['f'][y,x]:.4g}")
