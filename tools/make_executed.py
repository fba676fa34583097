"""Build executed.json / traffic.json entries from one round_profile.sh
output directory (ncu --set full summaries of the stage kernels), stamped
with the source hash of the library that was profiled.  bench.py reads
profiles/executed.json and refuses entries whose stamp differs from the
current sources (roofline.executed_frac = null then).
Usage: python tools/make_executed.py gpurun_out/<dir>  (writes <dir>/executed.json, traffic.json)"""
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__ as ge  # noqa: E402

d = sys.argv[1]
stamp = ge.source_hash()
so = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1702_07482_b200", "libtnrd.so")
import hashlib  # noqa: E402
so_hash = hashlib.sha1(open(so, "rb").read()).hexdigest()[:16] if os.path.exists(so) else None
ex = {"_note": ("Executed work of the dominant stage kernel per pixel-stage from ncu --set full SASS "
                "counts (tools/ncu_sass_stats.py; thread FMA = (FFMA + 2 FFMA2) warp instructions x 32 "
                "per pixel of one launch).  bench.py multiplies 2 FLOP x fma_per_px_stage by the live "
                "launch time into roofline.executed_frac, only when source_hash matches the library "
                "it runs."),
      "source_hash": stamp, "libtnrd_sha1": so_hash}
tr = {"_note": "dram__bytes_read.sum + dram__bytes_write.sum of one launch of the dominant stage kernel "
               "(ncu --set full), bytes", "source_hash": stamp}
for cfg, name in (("c1", "c1_cluster"), ("c2", "c2_cluster"), ("c3", "c3_tile"), ("c4", "c4_tile"), ("c5", "c5_tile")):
    p = os.path.join(d, f"ncu_summary_{name}.txt")
    if not os.path.exists(p):
        continue
    t = open(p).read()
    m = re.search(r"warp instr per pixel-stage (\d+): (.*)", t)
    if not m:
        continue
    ops = dict((k, float(v)) for k, v in re.findall(r"(\w+)=([\d.]+)", m.group(2)))
    fma = 32.0 * (ops.get("FFMA", 0.0) + 2.0 * ops.get("FFMA2", 0.0))

    def metric(label):
        mm = re.search(rf"{re.escape(label)}\s+([\d.]+)\s*(\S*)", t)
        if not mm:
            return None
        v, u = float(mm.group(1)), mm.group(2)
        scale = {"Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9, "byte": 1.0}.get(u, 1.0)
        return v * scale
    kern = re.search(r"== (.*)", t).group(1)[:80]
    ex[cfg] = {"kernel": kern, "ffma_per_px_stage": round(fma),
               "warp_instr_per_px_stage": int(m.group(1)),
               "issue_active": round(metric("issue active %") / 100, 3),
               "fma_pipe_instr": round(metric("FMA pipe %") / 100, 3),
               "source": f"profiles/<round>/ncu_summary_{name}.txt", "source_hash": stamp}
    rd, wr = metric("dram read"), metric("dram write")
    if rd is not None and wr is not None:
        tr[cfg] = rd + wr
json.dump(ex, open(os.path.join(d, "executed.json"), "w"), indent=1)
json.dump(tr, open(os.path.join(d, "traffic.json"), "w"), indent=1)
print(json.dumps(ex, indent=1))
print(json.dumps(tr, indent=1))
