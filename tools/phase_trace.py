"""Per-phase share of the tile kernel's CTA time (a -DTNRD_PHASE_TRACE build:
tools/build_variant.sh phase -DTNRD_PHASE_TRACE; TNRD_LIB_PATH=build_variants/libtnrd_phase.so).
Thread 0 of each CTA adds the clocks between the phase barriers to global
totals: staging | forward + RBF | phi fix-up | backward | epilogue.
Usage: python tools/phase_trace.py [c3|c5|c2] [batch]"""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1702_07482_b200 as tn
from paper_1702_07482_b200 import _lib, synth

key = sys.argv[1] if len(sys.argv) > 1 else "c3"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 32
mode = int(sys.argv[3]) if len(sys.argv) > 3 else 4
cfg = synth.CONFIGS[key]
model = synth.config_model(cfg)
dm = tn.device_model_for(model)
nb = min(B, 16)
base = torch.from_numpy(synth.noisy_batch(cfg, range(nb))).cuda()
f = base.repeat((B + nb - 1) // nb, 1, 1)[:B].contiguous()
out = torch.empty_like(f); work = torch.empty_like(f)
L = _lib.load()
L.tnrd_phase_trace.restype = ctypes.c_int
buf = (ctypes.c_ulonglong * 8)()
_lib.set_stage_kernel(mode)
for _ in range(2): dm.despeckle(f, out=out, work=work, check=False)
L.tnrd_phase_trace(buf)   # clear
dm.despeckle(f, out=out, work=work, check=False)
L.tnrd_phase_trace(buf)
v = np.array(list(buf), dtype=np.float64)
tot = v[:5].sum()
names = ["staging", "forward+RBF", "phi fix-up", "backward", "epilogue"]
print(f"{key} B={B} mode {mode}: {int(v[5])} CTAs, {tot / v[5]:.0f} clocks per CTA")
for n, x in zip(names, v[:5]):
    print(f"  {n:12s} {100 * x / tot:5.1f}%   {x / v[5]:9.0f} clocks per CTA")
