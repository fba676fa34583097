"""Per-CTA timeline of the split stage kernel (build with -DTNRD_SPLIT_TRACE,
load through TNRD_LIB_PATH): SM, start/end (globaltimer) and units per CTA of
the last launch.  Usage: TNRD_LIB_PATH=... python tools/split_trace.py MODE"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1702_07482_b200 as tn  # noqa: E402
from paper_1702_07482_b200 import _lib, synth  # noqa: E402

mode = int(sys.argv[1]) if len(sys.argv) > 1 else 6
key = sys.argv[2] if len(sys.argv) > 2 else "c2"
_lib.set_stage_kernel(mode)
cfg = synth.CONFIGS[key]
model = synth.config_model(cfg)
f = torch.from_numpy(synth.noisy_image(cfg, 0)[1]).cuda()
dm = tn.device_model_for(model)
for _ in range(3):
    dm.despeckle(f)
torch.cuda.synchronize()
L = _lib.load()
buf = (ctypes.c_ulonglong * (4096 * 4))()
L.tnrd_debug_split_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert L.tnrd_debug_split_trace(buf, 4096) == 0
a = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 4).astype(np.int64)
a = a[a[:, 1] > 0]
first = a[:, 3] >> 32
a[:, 3] &= 0xffffffff
np.save(os.environ.get("TRACE_OUT", "/tmp/trace.npy"), np.c_[a, first])
t0 = a[:, 1].min()
st, en, sm, un = (a[:, 1] - t0) / 1e3, (a[:, 2] - t0) / 1e3, a[:, 0], a[:, 3]
print(f"{key} mode {mode}: {len(a)} CTAs, kernel span {en.max():.1f} us; start spread {st.max():.1f} us")
print("units per CTA:", np.bincount(un))
print("CTA end times (us) pct 0/10/50/90/100:", np.percentile(en, [0, 10, 50, 90, 100]).round(1))
per_sm_end = {}
per_sm_units = {}
for s_, e_, u_ in zip(sm, en, un):
    per_sm_end[s_] = max(per_sm_end.get(s_, 0), e_)
    per_sm_units[s_] = per_sm_units.get(s_, 0) + u_
ends = np.array(list(per_sm_end.values()))
us = np.array(list(per_sm_units.values()))
print("SM last-end pct 0/10/50/90/100:", np.percentile(ends, [0, 10, 50, 90, 100]).round(1))
print("units per SM:", np.bincount(us))
busy = sum(e - s for s, e in zip(st, en))
print(f"CTA-busy fraction of span x CTAs: {busy / (en.max() * len(a)):.3f}")
print("us per unit (median over CTAs):", np.median((en - st) / np.maximum(un, 1)).round(2))
