#!/usr/bin/env python
"""Benchmark of the B200 TNRD despeckling path (contract: DESIGN.md §5).

    python bench.py [--gpus N] [--steps K] [--warmup W]
                    [--workload c1|c2|c3|c4|c5] [--impl ours|reference]

A step = one full despeckle (T fused stages) of one batch of the workload.
Default workload = C3 (BASELINE.json configs[2]): 256 images of 512x512,
7x7, Nk=48, T=5 -- the batch the metric quotes "at 1/2/4/8 B200", sharded
over the ranks (strong scaling, no data-path collective).  C4 splits one
16384^2 scene into row strips with a per-stage halo exchange (NCCL P2P);
C1/C2 are single images (replicas, one per rank); C5 is the 9x9 / Nk=80 /
T=8 batch.  Under torchrun every rank despeckles its shard; rank 0 prints
ONE JSON line.  At N > 1 the line carries `verify`: every rank's per-image
(per-strip) output hashes against rank 0's N = 1 recomputation of the whole
workload after the timed region.

--impl reference times the reference's CPU algorithm: the reference is pure
Python/numpy and cannot travel to the GPU box, so the float64 C port in
oracle/ (pinned to the reference's golden vectors, tests/test_oracle.py)
runs with every host thread on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import ctypes
import hashlib
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = ("megapixels/sec for full TNRD despeckle (7×7, 48 filters, "
          "5 stages) at 1/2/4/8 B200")
UNIT = "MPix/s"
DEFAULT_WORKLOAD = "c3"
DEFAULT_STEPS = {"c1": 200, "c2": 200, "c3": 20, "c4": 5, "c5": 10}


def w_contraction(cfg) -> int:
    """FLOP per pixel-stage of the two 49x48 contractions the direct method
    cannot skip: forward filter bank + adjoint, Nk m^2 FMA each (FMA = 2)."""
    return 4 * cfg.nk * cfg.m * cfg.m


def w_flop(cfg) -> int:
    """algorithmic FLOP per pixel-stage (FMA = 2), charging
    M = 63 Gaussian terms per response."""
    return 4 * cfg.nk * cfg.m * cfg.m + 5 * cfg.nk * cfg.M + 10


def w_sfu(cfg) -> int:
    return cfg.nk * cfg.M + 2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--_cpu-worker", dest="cpu_worker", default=None, help=argparse.SUPPRESS)
    a = ap.parse_args()
    if a.steps is None:
        a.steps = DEFAULT_STEPS[a.workload]
    return a


# Functional check of the N > 1 code path on a one-GPU box: every rank on
# cuda:0, gloo for the barriers, reductions and C4's (host-staged) halo
# exchange.  Not a measurement (ranks share the SMs); the line says so.
SHARED_GPU = os.environ.get("TNRD_BENCH_SHARED_GPU") == "1"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if SHARED_GPU:
        local = 0
    return rank, world, local


# ---------------------------------------------------------------- clocks

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.15)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.05)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- CPU baseline
# The reference's algorithm on the host cores: the float64 C port in oracle/
# (test infrastructure; used here only as the reported baseline).

def host_info() -> dict:
    """CPU model, logical cores and RAM of this host."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    ram = None
    try:
        ram = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 2 ** 30
    except (ValueError, OSError):
        pass
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(),
            "ram_gib": round(ram, 1) if ram else None}


def _crop(cfg, index: int, side: int) -> np.ndarray:
    """A centred side x side crop of workload image `index` (C4: of the
    scene's first tile row), float64."""
    from paper_1702_07482_b200 import synth
    if cfg.tiled:
        y0 = (1024 - side) // 2 + 1024 * (index % 16)
        x0 = (1024 - side) // 2 + 1024 * ((index // 16) % 16)
        return synth.scene_crop(cfg, y0, y0 + side, x0, x0 + side).astype(np.float64)
    _, f = synth.noisy_image(cfg, index % cfg.batch)
    y0, x0 = (cfg.H - side) // 2, (cfg.W - side) // 2
    return f[y0:y0 + side, x0:x0 + side].astype(np.float64)


def cpu_worker(spec: str) -> None:
    """Subprocess body (--_cpu-worker JSON): run the C port on one crop and
    print {seconds, t_end, peak_rss_mb}; `start` = a wall-clock time to wait
    for (so P workers start together)."""
    import resource
    a = json.loads(spec)
    from oracle import oracle as O
    from paper_1702_07482_b200 import synth
    cfg = synth.CONFIGS[a["workload"]]
    model = synth.config_model(cfg)
    crop = _crop(cfg, a["index"], a["side"])
    O.build()
    O.set_threads(a["threads"])
    while time.time() < a.get("start", 0):
        time.sleep(0.001)
    t0 = time.perf_counter()
    O.run_diffusion(crop, model)
    dt = time.perf_counter() - t0
    # VmHWM (this process image's high-water mark): ru_maxrss would carry
    # the forking parent's RSS across exec
    hwm = None
    with open("/proc/self/status") as fh:
        for line in fh:
            if line.startswith("VmHWM:"):
                hwm = float(line.split()[1]) / 1024.0
    if hwm is None:
        hwm = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1024.0
    print(json.dumps({"seconds": dt, "t_end": time.time(), "peak_rss_mb": hwm}))


def _spawn_worker(workload, index, side, threads, start=0.0):
    spec = json.dumps({"workload": workload, "index": index, "side": side,
                       "threads": threads, "start": start})
    return subprocess.Popen([sys.executable, os.path.join(REPO, "bench.py"), "--_cpu-worker", spec],
                            stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True, cwd=REPO)


def _collect(p):
    out, err = p.communicate()
    if p.returncode != 0:
        raise RuntimeError(f"cpu worker failed: {err[-500:]}")
    return json.loads(out.strip().splitlines()[-1])


def cpu_all_threads(cfg, budget_s: float):
    """The C port with every host thread on image 0 of the workload (a
    centred crop, shrunk until one run fits budget_s).  Returns (MPix/s,
    seconds, side, threads, peak_rss_mb)."""
    from oracle import oracle as O
    O.build()
    O.set_threads(-1)
    threads = O.threads()
    side = min(cfg.H, cfg.W, 1024)
    while True:
        r = _collect(_spawn_worker(cfg.name, 0, side, -1))
        if r["seconds"] <= budget_s or side <= 64:
            break
        side = max(64, int(side * (budget_s / r["seconds"]) ** 0.5 * 0.9) // 8 * 8)
    return side * side / r["seconds"] / 1e6, r["seconds"], side, threads, r["peak_rss_mb"]


def cpu_baseline(cfg) -> dict:
    """SURVEY 8(d)'s CPU figures for the line: all host threads on one image
    (the value), one core (extrapolated to a full image), P single-threaded
    processes on P different images at once (image-parallel throughput),
    and peak RSS."""
    info = host_info()
    rate, dt, side, threads, rss = cpu_all_threads(cfg, 20.0)
    full = side == min(cfg.H, cfg.W) and cfg.H == cfg.W and not cfg.tiled
    out = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
           "sample": (f"{side}x{side} {'(full image)' if full else 'centred crop'} of image 0, "
                      f"{cfg.m}x{cfg.m}, Nk={cfg.nk}, T={cfg.T}, float64 C port of the reference "
                      f"algorithm (oracle/tnrd_oracle.c), {threads} threads"),
           "peak_rss_mb": round(rss, 1), **info}
    # one core: a small crop, extrapolated per pixel-stage to one full image
    cs = 128 if cfg.m <= 7 else 96
    r1 = _collect(_spawn_worker(cfg.name, 0, cs, 1))
    per_px = r1["seconds"] / (cs * cs)
    out["single_core"] = {
        "value": cs * cs / r1["seconds"] / 1e6, "unit": UNIT, "cores": 1,
        "sample": f"{cs}x{cs} centred crop of image 0, 1 thread",
        "full_image_seconds_extrapolated": per_px * cfg.H * cfg.W,
        "note": f"extrapolated per pixel from the {cs}x{cs} crop to one {cfg.H}x{cfg.W} image",
        "peak_rss_mb": round(r1["peak_rss_mb"], 1)}
    # P processes x 1 thread, each on its own image (the reference's natural
    # parallelism: images are independent)
    P = os.cpu_count() or 1
    start = time.time() + 1.5
    procs = [_spawn_worker(cfg.name, i, cs, 1, start) for i in range(P)]
    res = [_collect(p) for p in procs]
    wall = max(r["t_end"] for r in res) - start
    out["image_parallel"] = {
        "value": P * cs * cs / wall / 1e6, "unit": UNIT, "processes": P, "cores": P,
        "sample": f"{P} processes x 1 thread, each a {cs}x{cs} crop of its own image, started together",
        "peak_rss_mb_per_process": round(max(r["peak_rss_mb"] for r in res), 1),
        "note": ("the reference's numpy path materialises the (Nk,H,W,M) RBF design tensor: "
                 "SURVEY 8(d) measured ~6.4 GB RSS per 512^2 image for C2/C3 (~42 GB for C5), "
                 "which caps P at RAM/RSS for the reference itself; the C port streams it")}
    return out


def run_reference_arm(args, cfg, rank):
    if rank != 0:
        return
    from paper_1702_07482_b200 import synth
    model = synth.config_model(cfg)
    per_step = max(2.0, 150.0 / max(1, args.steps + args.warmup))
    rate, dt, side, threads, rss = cpu_all_threads(cfg, per_step)
    from oracle import oracle as O
    O.set_threads(-1)
    crop = _crop(cfg, 0, side)
    for _ in range(max(0, args.warmup - 1)):
        O.run_diffusion(crop, model)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.run_diffusion(crop, model)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * sum(times) / len(times)
    value = side * side / (ms * 1e3)
    sample = (f"{side}x{side} centred crop of image 0 per step, {cfg.m}x{cfg.m}, Nk={cfg.nk}, "
              f"T={cfg.T}, float64 C port of the reference algorithm (oracle/tnrd_oracle.c), "
              f"{threads} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(cfg, args, per_rank_batch=1),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads,
                         "kind": "port", "sample": sample, "peak_rss_mb": round(rss, 1),
                         **host_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- ours

def workload_config(cfg, args, per_rank_batch):
    return {
        "workload": f"{cfg.name}: {cfg.note}",
        "H": cfg.H, "W": cfg.W, "filter_size": cfg.m, "num_filters": cfg.nk,
        "stages": cfg.T, "rbf_centres": cfg.M, "images_per_rank": per_rank_batch,
        "parallelism": f"{'replicas' if cfg.batch == 1 else 'batch-sharded'} x{args.gpus}",
        "l2": "256 MiB L2-flush write between timed steps, outside the per-step CUDA events",
        "inputs": "seeded piecewise-smooth clean x Philox amplitude speckle (synth.py)",
    }


def measure_peaks(torch, L, stream):
    """FFMA (TFLOP/s) and MUFU ex2 (Gop/s) peaks measured on this GPU."""
    out = {}
    for kind, key in ((0, "fp32_tflops"), (1, "mufu_ex2_gops")):
        ops = ctypes.c_double(0)
        iters = 20000 if kind == 0 else 8000
        for _ in range(2):
            L.tnrd_probe(kind, iters, 4, ctypes.c_void_p(stream.cuda_stream), ctypes.byref(ops))
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        best = 0.0
        for _ in range(3):
            e0.record(stream)
            L.tnrd_probe(kind, iters, 4, ctypes.c_void_p(stream.cuda_stream), ctypes.byref(ops))
            e1.record(stream)
            e1.synchronize()
            best = max(best, ops.value / (e0.elapsed_time(e1) * 1e-3))
        out[key] = best / (1e12 if kind == 0 else 1e9)
    return out


def shard_indices(cfg, rank, world):
    if cfg.batch == 1:
        return [rank]                     # C1/C2: one image per rank (replicas)
    per = cfg.batch // world              # C3/C5: batch sharded (strong)
    return list(range(rank * per, (rank + 1) * per))


def img_hash(a: np.ndarray) -> str:
    return hashlib.sha1(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()[:16]


def stamp_ok(entry) -> tuple[bool, str]:
    """executed.json entries are stamped with the hash of the sources the
    profiled library was built from (__graft_entry__.source_hash)."""
    import __graft_entry__ as ge
    cur = ge.source_hash()
    got = entry.get("source_hash")
    if got == cur:
        return True, cur
    return False, f"stale: profiled build {got}, this build {cur}"


def main():
    args = parse()
    if args.cpu_worker is not None:
        cpu_worker(args.cpu_worker)
        return
    rank, world, local = dist_env()
    from paper_1702_07482_b200 import synth
    cfg = synth.CONFIGS[args.workload]
    if args.impl == "reference":
        run_reference_arm(args, cfg, rank)
        return

    # inputs first (host cores, before any CUDA work in this process)
    if cfg.name == "c4":
        from paper_1702_07482_b200 import strips
        lay = strips.StripLayout(cfg.H, cfg.W, world, rank, halo=cfg.m - 1)
        r0, r1 = lay.rows
        f_host = synth.scene_rows_parallel(cfg, r0, r1)[None]
        idx = None
    else:
        idx = shard_indices(cfg, rank, world)
        f_host = synth.noisy_batch(cfg, idx)

    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if SHARED_GPU:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_1702_07482_b200 as tn
    from paper_1702_07482_b200 import _lib, strips

    L = _lib.load()
    model = synth.config_model(cfg)
    dm = tn.device_model_for(model)
    dev = torch.device("cuda", local)
    red_dev = torch.device("cpu") if SHARED_GPU else dev   # max-over-ranks reductions
    stream = torch.cuda.Stream(dev)
    status = tn.engine.Status(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    H, W = cfg.H, cfg.W
    sh = ctypes.c_void_p(stream.cuda_stream)
    sptr = ctypes.c_void_p(status.buf.data_ptr())

    if cfg.name == "c4":
        # one scene split into row strips, per-stage halo exchange (NCCL P2P;
        # host-staged gloo when the ranks share one GPU)
        h, n = lay.halo, lay.n
        f_ext = torch.zeros(n + 2 * h, W, dtype=torch.float32, device=dev)
        f_ext[h:h + n] = torch.from_numpy(f_host[0]).to(dev)
        bufs = [torch.empty_like(f_ext), torch.empty_like(f_ext)]
        stage_fn = strips.gpu_stage_fn(dm, status=status, stream=stream)
        if world == 1:
            exch = lambda *a, **k: None  # noqa: E731
        else:
            exch = strips.exchange_halos_host if SHARED_GPU else strips.exchange_halos
        B, px_rank = 1, n * W
        result = {}

        def step(evs=None):
            L.tnrd_status_reset(sptr, sh)
            if evs is not None:
                evs[0].record(stream)
            exch(f_ext, lay)
            cur = f_ext
            for t in range(cfg.T):
                if t > 0:
                    exch(cur, lay)
                if evs is not None and t > 0:
                    evs[t].record(stream)
                dst = bufs[t % 2]
                fl = lay.flags | ((_lib.STAGE_FLOOR_INPUT | _lib.STAGE_CHECK_F) if t == 0 else 0)
                stage_fn(t, cur, f_ext, dst, lay, fl)
                cur = dst
            if evs is not None:
                evs[cfg.T].record(stream)
            result["u"] = cur

        def final_output():
            return result["u"][h:h + n]
    else:
        B = len(idx)
        f = torch.from_numpy(f_host).to(dev)
        out = torch.empty_like(f)
        work = torch.empty_like(f)
        px_rank = B * H * W

        def step(evs=None):
            # T fused stage launches through the C ABI; final stage lands in `out`
            L.tnrd_status_reset(sptr, sh)
            if B >= 2:
                # batches: one tnrd_despeckle call, which may run the two
                # halves' stage chains on two streams (DESIGN.md §7b item 5);
                # events bracket the whole step, per-stage time = step / T
                if evs is not None:
                    evs[0].record(stream)
                _lib.check(L.tnrd_despeckle(dm.handle, ctypes.c_void_p(f.data_ptr()),
                                            ctypes.c_void_p(out.data_ptr()),
                                            ctypes.c_void_p(work.data_ptr()),
                                            B, H, W, W, H * W, sptr, sh))
                if evs is not None:
                    evs[cfg.T].record(stream)
                return
            cur = f
            for t in range(cfg.T):
                dst = out if (cfg.T - 1 - t) % 2 == 0 else work
                fl = (_lib.STAGE_FLOOR_INPUT | _lib.STAGE_CHECK_F) if t == 0 else 0
                if evs is not None:
                    evs[t].record(stream)
                rc = L.tnrd_stage(dm.handle, t, ctypes.c_void_p(cur.data_ptr()),
                                  ctypes.c_void_p(f.data_ptr()), ctypes.c_void_p(dst.data_ptr()),
                                  B, H, W, W, H * W, fl, sptr, sh)
                if rc:
                    _lib.check(rc)
                cur = dst
            if evs is not None:
                evs[cfg.T].record(stream)

        def final_output():
            return out

    with torch.cuda.stream(stream):
        for _ in range(max(3, args.warmup)):
            step()
            flush.zero_()
        stream.synchronize()
        status.check()
        peaks = measure_peaks(torch, L, stream)
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        smi_index = int(vis.split(",")[local]) if vis and vis.split(",")[local].isdigit() else local
        clocks = ClockSampler(smi_index)
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(cfg.T + 1)]
               for _ in range(args.steps)]
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)
        clocks.start()
        _lib.launch_count_reset()
        for k in range(args.steps):
            step(evs[k])
            flush.zero_()                 # outside the events: L2 flush
        torch.cuda.synchronize(dev)
        launches = _lib.launch_count()
        if dist is not None:
            dist.barrier()
        clk = clocks.stop()
        status.check()
        out_host = final_output().cpu().numpy()

    step_ms = [evs[k][0].elapsed_time(evs[k][cfg.T]) for k in range(args.steps)]
    ms = sum(step_ms) / len(step_ms)
    if cfg.name == "c4" or px_rank > H * W:
        # C4: stage launches interleave with halo exchanges; batches: one
        # tnrd_despeckle call per step -- per-launch time = step / T
        launch_ms = ms / cfg.T
    else:
        stage_ms = [evs[k][t].elapsed_time(evs[k][t + 1])
                    for k in range(args.steps) for t in range(cfg.T)]
        launch_ms = sum(stage_ms) / len(stage_ms)
    if dist is not None:
        tt = torch.tensor([ms, launch_ms], device=red_dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms, launch_ms = tt.tolist()
    total_px = world * px_rank if cfg.name != "c4" else H * W
    value = total_px / (ms * 1e3)          # MPix/s, all ranks

    # ---- e2e: HOST buffers in, HOST result out, copies inside the timed region
    e2e_steps, e2e_same = 0, None
    if cfg.name == "c4" and world == 1:
        # the whole scene through tnrd_plan_despeckle_host (C ABI): row bands
        # on their own streams, each band's H2D / stages / D2H ordered by
        # events only where the data flows, so the copies overlap the stages
        pin_f = torch.from_numpy(f_host[0]).pin_memory()
        pin_u = torch.empty_like(pin_f).pin_memory()
        plan = dm._plan(1, H, W)
        pstream = torch.cuda.ExternalStream(L.tnrd_plan_stream(plan), device=dev)

        def run_scene():
            _lib.check(L.tnrd_plan_despeckle_host(plan, ctypes.c_void_p(pin_f.data_ptr()),
                                                  ctypes.c_void_p(pin_u.data_ptr())))

        run_scene()
        e2e_steps = max(2, min(args.steps, 5))
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        e0.record(pstream)
        for _ in range(e2e_steps):
            run_scene()
        e1.record(pstream)
        e1.synchronize()
        e2e_ms = e0.elapsed_time(e1) / e2e_steps
        e2e_same = bool(np.array_equal(pin_u.numpy(), out_host))
        e2e_path = ("tnrd_plan_despeckle_host (C ABI), one scene per step: row bands with "
                    "event-ordered H2D / stages / D2H on their own streams, pinned host buffers")
    elif cfg.name == "c4":
        pin_f = torch.from_numpy(f_host[0]).pin_memory()
        pin_u = torch.empty_like(pin_f).pin_memory()
        e2e_steps = max(2, min(args.steps, 5))
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            if dist is not None:
                dist.barrier()
            torch.cuda.synchronize(dev)
            e0.record(stream)
            for _ in range(e2e_steps):
                f_ext[h:h + n].copy_(pin_f, non_blocking=True)
                step()
                pin_u.copy_(final_output(), non_blocking=True)
                status.check()
            e1.record(stream)
            e1.synchronize()
        e2e_ms = e0.elapsed_time(e1) / e2e_steps
        e2e_path = "strip H2D + run_strip (halo exchange, fused stages) + D2H + status check"
    else:
        plan = dm._plan(B, H, W)
        pstream = torch.cuda.ExternalStream(L.tnrd_plan_stream(plan), device=dev)
        per_img = int(f_host.nbytes)
        # a stream of steps through tnrd_plan_despeckle_host_many: every step
        # still copies its input in and its result out (pinned buffers), and
        # one step's copies overlap the next step's stages
        # (enough steps that the first copy-in and the last copy-out, which
        # nothing overlaps, are a small share: <= 2 GiB of pinned input)
        e2e_steps = max(3, min(args.steps, 50, max(2, (2048 << 20) // per_img)))
        seq_f = torch.empty((e2e_steps,) + tuple(f_host.shape), dtype=torch.float32).pin_memory()
        seq_f.copy_(torch.from_numpy(f_host).unsqueeze(0).expand_as(seq_f))
        seq_u = torch.empty_like(seq_f).pin_memory()
        bad = ctypes.c_int(-1)

        def run_many():
            _lib.check(L.tnrd_plan_despeckle_host_many(
                plan, ctypes.c_void_p(seq_f.data_ptr()), ctypes.c_void_p(seq_u.data_ptr()),
                e2e_steps, ctypes.byref(bad)))

        run_many()   # warm-up: twin plans, graphs
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        if dist is not None:
            dist.barrier()
        e0.record(pstream)
        run_many()
        e1.record(pstream)
        e1.synchronize()
        e2e_ms = e0.elapsed_time(e1) / e2e_steps
        e2e_path = ("tnrd_plan_despeckle_host_many (C ABI): a stream of steps, each with its "
                    "H2D + T stages + D2H + status read, pinned host buffers")
        e2e_same = all(bool(np.array_equal(seq_u[k].numpy(), out_host)) for k in range(e2e_steps))
        del seq_f, seq_u
    if dist is not None:
        tt = torch.tensor([e2e_ms], device=red_dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = tt.item()

    # ---- N > 1: every rank's output against rank 0's N = 1 recomputation
    verify = None
    if dist is not None and not args.no_verify:
        if cfg.name == "c4":
            mine = [(r0, r1, img_hash(out_host))]
        else:
            mine = [(i, img_hash(out_host[j])) for j, i in enumerate(idx)]
        got = [None] * world
        dist.all_gather_object(got, mine)
        if rank == 0:
            t0 = time.perf_counter()
            if cfg.name == "c4":
                whole = synth.scene_rows_parallel(cfg, 0, H)
                u1 = dm.despeckle(torch.from_numpy(whole).to(dev)).cpu().numpy()
                items = [x for part in got for x in part]
                bad_items = [(a, b) for a, b, hsh in items if img_hash(u1[a:b]) != hsh]
                what = f"{len(items)} strips"
            else:
                # rank 0 recomputes every rank's shard as its own call (the
                # stage kernel, and with it the summation order, is chosen
                # from the launch's grid size, so a shard's bits are those of
                # a same-sized N = 1 call) and, as one call, the whole batch
                # (agreement to fp32 summation order)
                all_idx = [x[0] for part in got for x in part]
                fb = torch.from_numpy(synth.noisy_batch(cfg, all_idx)).to(dev)
                if cfg.batch == 1:
                    u1 = np.stack([dm.despeckle(fb[j]).cpu().numpy() for j in range(len(all_idx))])
                    whole_rel = 0.0
                else:
                    parts, j0 = [], 0
                    for part in got:
                        parts.append(dm.despeckle(fb[j0:j0 + len(part)]).cpu().numpy())
                        j0 += len(part)
                    u1 = np.concatenate(parts)
                    uw = dm.despeckle(fb).cpu().numpy()
                    whole_rel = float(np.max(np.abs(u1 - uw) / np.abs(uw)))
                    del uw
                ref = {i: img_hash(u1[j]) for j, i in enumerate(all_idx)}
                items = [x for part in got for x in part]
                bad_items = [i for i, hsh in items if ref[i] != hsh]
                if whole_rel > 1e-5:
                    bad_items.append(f"whole-batch call differs by {whole_rel:.2e}")
                what = f"{len(items)} images"
            verify = {"ok": not bad_items, "checked": what, "mismatches": bad_items[:8],
                      "how": ("sha1 of each rank's fp32 output (per image / per strip) vs rank 0 "
                              "recomputing it after the timed region: batches shard by shard (same "
                              "grid size, hence same kernel and bits) plus the whole batch in one call "
                              "(max relative difference <= 1e-5, fp32 summation order); C4 as the whole scene"),
                      "seconds": round(time.perf_counter() - t0, 2)}
        dist.barrier()

    # ---- latency: one image through a fresh one-image plan, host to host
    latency = None
    if rank == 0:
        lat_img = f_host[0]
        pin_f1 = torch.from_numpy(np.ascontiguousarray(lat_img)).pin_memory()
        pin_u1 = torch.empty_like(pin_f1).pin_memory()
        plan1 = dm._plan(1, lat_img.shape[0], lat_img.shape[1])
        lat = []
        reps = 3 if lat_img.size > (1 << 22) else 20
        for k in range(reps + 2):
            t0 = time.perf_counter()
            _lib.check(L.tnrd_plan_despeckle_host(plan1, ctypes.c_void_p(pin_f1.data_ptr()),
                                                  ctypes.c_void_p(pin_u1.data_ptr())))
            if k >= 2:
                lat.append(time.perf_counter() - t0)
        lms = 1e3 * statistics.median(lat)
        latency = {"ms": lms, "value": lat_img.size / (lms * 1e3), "unit": UNIT,
                   "image": f"{lat_img.shape[0]}x{lat_img.shape[1]}",
                   "path": ("tnrd_plan_despeckle_host (C ABI), one image, one plan, pinned host "
                            "buffers, no overlap: host wall clock around H2D + T stages + D2H + "
                            f"status read, median of {reps}")}

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (the fused stage)
    stage_kernels = int(round(launches / (args.steps * cfg.T)))
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    half_tiles = -(-H // 64) * -(-W // 64) * (px_rank // (H * W) // 2)
    forked = (cfg.name != "c4" and px_rank > H * W and half_tiles >= 3 * 2 * sms
              and os.environ.get("TNRD_BATCH_FORK", "1")[:1] != "0")
    if forked and stage_kernels == 2:
        stage_kernels = "stage_kernel_pt (fused tile kernel) x 2 batch halves on two streams"
    else:
        tiles_rank = -(-H // 64) * -(-W // 64) * (px_rank // (H * W))
        one = ("stage_kernel_pt (fused tile kernel)" if tiles_rank >= 2 * 3 * 2 * sms else
               "stage_kernel_cl_pt (fused cluster kernel: a tile's filter groups on the CTAs of a "
               "thread-block cluster, partial forces summed through distributed shared memory)")
        if cfg.name == "c1":
            one = one.replace("stage_kernel_cl_pt", "stage_kernel_cl")
        stage_kernels = {1: one,
                         2: "stage_kernel_split_pt + stage_reduce_kernel"}.get(stage_kernels,
                                                                                 str(stage_kernels))
    px_launch = px_rank
    peak_tf = peaks["fp32_tflops"]
    contraction_tf = w_contraction(cfg) * px_launch / (launch_ms * 1e-3) / 1e12
    alg_tf = w_flop(cfg) * px_launch / (launch_ms * 1e-3) / 1e12
    peak_sfu = peaks["mufu_ex2_gops"] * 1e9
    t_roof = max(w_flop(cfg) / (peak_tf * 1e12), w_sfu(cfg) / peak_sfu)  # s per pixel-stage
    roof_pxst = 1.0 / t_roof / 1e6                                        # MPix*stages/s
    ach_pxst = px_launch / (launch_ms * 1e-3) / 1e6
    traffic = None
    tpath = os.path.join(REPO, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(cfg.name)
    # what the stage kernel executes (ncu --set full SASS counts of THIS
    # build, profiles/executed.json, stamped with the source hash) at this
    # run's live launch time
    executed, executed_frac = None, None
    epath = os.path.join(REPO, "profiles", "executed.json")
    if os.path.exists(epath):
        ex = json.load(open(epath)).get(cfg.name)
        if ex:
            ok, why = stamp_ok(ex)
            ex_tf = 2.0 * ex["ffma_per_px_stage"] * px_launch / (launch_ms * 1e-3) / 1e12
            executed = dict(ex, achieved_tflops=ex_tf, stamp=why if not ok else "current build")
            executed_frac = ex_tf / peak_tf if ok else None
    conf = workload_config(cfg, args, B)
    if cfg.name == "c4":
        conf.update({"parallelism": (f"row strips x{world}, {cfg.m - 1}-row u halo exchanged per "
                                     f"stage ({'gloo host-staged' if SHARED_GPU else 'NCCL P2P'})"),
                     "rows_per_rank": px_rank // W})
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak" if cfg.batch == 1 and cfg.name != "c4" else "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": conf,
        "roofline": {
            "bound": "fp32", "unit": "TFLOP/s", "achieved": contraction_tf,
            "peak": peak_tf, "frac": contraction_tf / peak_tf, "traffic": traffic,
            "peak_source": "FFMA measured on this GPU by tnrd_probe; MEASURED_PEAKS.json has no FP32 entry",
            "work": (f"contraction FLOP the direct method cannot skip: 4*Nk*m^2 = {w_contraction(cfg)} "
                     f"per pixel-stage (forward + adjoint {cfg.m}x{cfg.m}x{cfg.nk} FMA) x {px_launch} "
                     "px per stage launch"),
            "launch_ms": launch_ms,
            "stage_kernels": stage_kernels,
            "executed_frac": executed_frac,
            "executed": executed,
            "algorithmic_frac": alg_tf / peak_tf,
            "algorithmic": {
                "note": (">1 by construction: SURVEY 8(d)'s W_flop charges 5*Nk*M FLOP of Gaussian "
                         "terms per pixel-stage, which the tabulated (cubic-interpolated) phi never "
                         "executes"),
                "w_flop": w_flop(cfg), "achieved_tflops": alg_tf,
                "survey_combined": {
                    "unit": "MPix*stages/s", "achieved": ach_pxst, "peak": roof_pxst,
                    "frac": ach_pxst / roof_pxst,
                    "rule": "t_roof = max(W_flop/P_fp32, W_sfu/P_mufu) with on-box P_fp32, P_mufu",
                    "p_mufu_gops": peaks["mufu_ex2_gops"]}},
        },
        "e2e": {"value": total_px / (e2e_ms * 1e3), "unit": UNIT,
                "h2d_bytes_per_step": int(f_host.nbytes),
                "d2h_bytes_per_step": int(f_host.nbytes) + 8,
                "steps": e2e_steps, "path": e2e_path,
                "same_bits_as_device_run": e2e_same},
        "e2e_latency": latency,
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if verify is not None:
        line["verify"] = verify
    if SHARED_GPU:
        line["not_a_measurement"] = (f"TNRD_BENCH_SHARED_GPU: {world} ranks shared cuda:0 "
                                     "(functional check of the N>1 path)")
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg)
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    if verify is not None and not verify["ok"]:
        sys.exit(3)


if __name__ == "__main__":
    main()
