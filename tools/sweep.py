"""Time build variants (TNRD_LIB_PATH) on C2 / C3-subset / C5-subset; one
process per variant so each loads its own library."""
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_1702_07482_b200 as tn
from paper_1702_07482_b200 import synth
from oracle import oracle as O
# parity spot check
cfg = synth.CONFIGS["c2"]; model = synth.config_model(cfg)
clean, f = synth.noisy_image(cfg, 0, 100, 90)
u, _ = tn.run_diffusion(f, model); ref = O.run_diffusion(f.astype(np.float64), model)
rel = float(np.max(np.abs(u - ref) / ref))
res = [f"rel={rel:.1e}"]
for key, B in (("c2", 1), ("c3", 32), ("c5", 4), ("c1", 1)):
    cfg = synth.CONFIGS[key]; model = synth.config_model(cfg)
    if key == "c5" and __import__("os").environ.get("TNRD_STAGE_KERNEL") == "2":
        continue
    f = torch.from_numpy(np.stack([synth.noisy_image(cfg, i)[1] for i in range(B)])).cuda()
    dm = tn.device_model_for(model)
    out = torch.empty_like(f); work = torch.empty_like(f)
    for _ in range(3): dm.despeckle(f, out=out, work=work, check=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    e0.record()
    for _ in range(n): dm.despeckle(f, out=out, work=work, check=False)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    res.append(f"{key}:{B * cfg.H * cfg.W * cfg.T / ms / 1e3:.0f}")
print(" ".join(res), "MPix*st/s")
''' % REPO

for arg in sys.argv[1:]:
    so, _, mode = arg.partition(":")
    env = dict(os.environ, TNRD_LIB_PATH=os.path.abspath(so))
    if mode:
        env["TNRD_STAGE_KERNEL"] = mode
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    print(f"{os.path.basename(so) + (':' + mode if mode else ''):26s}", (r.stdout.strip() or r.stderr.strip()[-300:]), flush=True)
