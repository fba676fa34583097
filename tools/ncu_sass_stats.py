"""Stall reasons, opcode mix (per pixel) and smem conflict hot spots of one
ncu report (source page, SASS)."""
import csv
import subprocess
import sys
from collections import Counter

path, px = sys.argv[1], float(sys.argv[2])
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[2:]


def f(r, k):
    try:
        return float(r[ix[k]] or 0)
    except (KeyError, ValueError):
        return 0.0


stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot_s = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data) or 1
agg = {h: sum(f(r, h) for r in data) for h in stalls}
print("stalls:", ", ".join(f"{k[6:]}={v / tot_s * 100:.0f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
c = Counter()
for r in data:
    src = r[ix["Source"]].split()
    if src:
        op = src[1] if src[0].startswith("@") else src[0]
        c[op.split(".")[0]] += f(r, "Instructions Executed")
print(f"warp instr per pixel-stage {sum(c.values()) / px:.0f}:",
      ", ".join(f"{k}={v / px:.1f}" for k, v in c.most_common(14)))
exc = sum(f(r, "L1 Wavefronts Shared Excessive") for r in data)
wf = sum(f(r, "L1 Wavefronts Shared") for r in data)
print(f"smem wavefronts/px {wf / px:.1f} (excess {exc / px:.1f})")
