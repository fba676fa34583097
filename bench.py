#!/usr/bin/env python
"""Benchmark of the B200 TNRD despeckling path (contract: see DESIGN.md §Bench).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|c3|c5]
                    [--impl ours|reference]

A step = one full despeckle (T fused stages) of one batch of the workload.
Default workload = BASELINE.json configs[1] (C2: one 512x512 image, 7x7,
Nk=48, T=5).  Under torchrun each rank despeckles its own image(s) (C2:
weak scaling, one image per rank; C3/C5: the batch split over ranks,
strong scaling); no data-path collective.  Rank 0 prints ONE JSON line.

--impl reference times the reference's CPU algorithm: the reference is pure
Python/numpy and cannot travel to the GPU box, so the float64 C port in
oracle/ (pinned bit-for-bit-ish to the reference's golden vectors, see
tests/test_oracle.py) runs with every host thread on a bounded sample of
the same workload.
"""
from __future__ import annotations

import argparse
import ctypes
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


def w_flop(cfg) -> int:
    """algorithmic FLOP per pixel-stage (FMA = 2)."""
    return 4 * cfg.nk * cfg.m * cfg.m + 5 * cfg.nk * cfg.M + 10


def w_sfu(cfg) -> int:
    return cfg.nk * cfg.M + 2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="c2", choices=["c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if SHARED_GPU:
        local = 0
    return rank, world, local


# Functional check of the N > 1 code path on a one-GPU box: every rank on
# cuda:0, gloo for the barriers and the max-over-ranks reductions.  Not a
# measurement (ranks share the SMs); the line says so.  C4's strip exchange
# needs NCCL and is not supported in this mode.
SHARED_GPU = os.environ.get("TNRD_BENCH_SHARED_GPU") == "1"


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

def host_info() -> dict:
    """CPU model and logical core count of this host (SURVEY 8(d) asks for
    both beside the CPU baseline)."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "os_cpu_count": os.cpu_count()}


def cpu_reference_run(cfg, model, f, budget_s: float):
    """Time the float64 C port of the reference algorithm (all host
    threads) on f, shrinking to a centred crop if a run exceeds budget_s.
    Returns (mpix_per_s, seconds, sample_desc, threads)."""
    from oracle import oracle as O
    O.build()
    O.set_threads(-1)
    threads = O.threads()
    H, W = f.shape
    side = min(H, W)
    while True:
        y0, x0 = (H - side) // 2, (W - side) // 2
        crop = f[y0:y0 + side, x0:x0 + side].astype(np.float64)
        t0 = time.perf_counter()
        O.run_diffusion(crop, model)
        dt = time.perf_counter() - t0
        if dt <= budget_s or side <= 64:
            break
        side = max(64, int(side * (budget_s / dt) ** 0.5 * 0.9) // 8 * 8)
    sample = (f"{side}x{side} crop of image 0 ({'full image' if side == min(H, W) and H == W else 'bounded sample'}), "
              f"{cfg.m}x{cfg.m}, Nk={cfg.nk}, T={cfg.T}, float64 C port of the reference "
              f"algorithm (oracle/tnrd_oracle.c), {threads} threads")
    return side * side / dt / 1e6, dt, sample, threads


def single_core_run(cfg, model, f, side: int = 128) -> dict:
    """SURVEY 8(d)'s 1-core figure: the same C port on one thread over a
    centred side x side crop (a few seconds)."""
    from oracle import oracle as O
    O.build()
    O.set_threads(1)
    try:
        H, W = f.shape
        y0, x0 = (H - side) // 2, (W - side) // 2
        crop = f[y0:y0 + side, x0:x0 + side].astype(np.float64)
        t0 = time.perf_counter()
        O.run_diffusion(crop, model)
        dt = time.perf_counter() - t0
    finally:
        O.set_threads(-1)
    return {"value": side * side / dt / 1e6, "unit": UNIT, "cores": 1,
            "sample": f"{side}x{side} centred crop of image 0, 1 thread"}


def run_reference_arm(args, cfg, rank):
    if rank != 0:
        return
    from paper_1702_07482_b200 import synth
    model = synth.config_model(cfg)
    if cfg.tiled:
        f = synth.scene_crop(cfg, 0, 1024, 0, 1024)
    else:
        _, f = synth.noisy_image(cfg, 0)
    per_step = max(2.0, 150.0 / max(1, args.steps + args.warmup))
    rate, dt, sample, threads = cpu_reference_run(cfg, model, f, per_step)
    from oracle import oracle as O
    side = int(round((rate * 1e6 * dt) ** 0.5))
    y0 = (f.shape[0] - side) // 2
    x0 = (f.shape[1] - side) // 2
    crop = f[y0:y0 + side, x0:x0 + side].astype(np.float64)
    for _ in range(max(0, args.warmup - 1)):
        O.run_diffusion(crop, model)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.run_diffusion(crop, model)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * sum(times) / len(times)
    value = side * side / (ms * 1e3)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(cfg, args, per_rank_batch=1),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads,
                         "kind": "port", "sample": sample, **host_info()},
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


def setup_images(cfg, rank, world):
    if cfg.batch == 1:
        idx = [rank]                      # C2: one image per rank (weak)
    else:
        per = cfg.batch // world          # C3/C5: batch sharded (strong)
        idx = list(range(rank * per, (rank + 1) * per))
    return idx, np.stack([synth_mod().noisy_image(cfg, i)[1] for i in idx])


def synth_mod():
    from paper_1702_07482_b200 import synth
    return synth


def main():
    args = parse()
    rank, world, local = dist_env()
    synth = synth_mod()
    cfg = synth.CONFIGS[args.workload]
    if args.impl == "reference":
        run_reference_arm(args, cfg, rank)
        return

    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if SHARED_GPU:
            assert cfg.name != "c4", "TNRD_BENCH_SHARED_GPU: C4 strips need NCCL"
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
        # one scene split into row strips, per-stage halo exchange (NCCL P2P)
        lay = strips.StripLayout(H, W, world, rank, halo=cfg.m - 1)
        r0, r1 = lay.rows
        h, n = lay.halo, lay.n
        f_host = synth.scene_rows(cfg, r0, r1)[None]
        f_ext = torch.zeros(n + 2 * h, W, dtype=torch.float32, device=dev)
        f_ext[h:h + n] = torch.from_numpy(f_host[0]).to(dev)
        bufs = [torch.empty_like(f_ext), torch.empty_like(f_ext)]
        stage_fn = strips.gpu_stage_fn(dm, status=status, stream=stream)
        exch = strips.exchange_halos if world > 1 else (lambda *a, **k: None)
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
        idx, f_host = setup_images(cfg, rank, world)
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
        e2e_path = "strip H2D + run_strip (NCCL halo exchange, fused stages) + D2H + status check"
    else:
        pin_f = torch.from_numpy(f_host).pin_memory()
        pin_u = torch.empty_like(pin_f).pin_memory()
        plan = dm._plan(B, H, W)
        pstream = torch.cuda.ExternalStream(L.tnrd_plan_stream(plan), device=dev)
        for _ in range(3):
            _lib.check(L.tnrd_plan_despeckle_host(plan, ctypes.c_void_p(pin_f.data_ptr()),
                                                  ctypes.c_void_p(pin_u.data_ptr())))
        # a stream of steps through tnrd_plan_despeckle_host_many: every step
        # still copies its input in and its result out (pinned buffers), and
        # one step's copies overlap the next step's stages
        per_img = int(f_host.nbytes)
        e2e_steps = max(3, min(args.steps, 50, max(2, (1 << 30) // per_img)))
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
        ref_u = final_output().cpu().numpy()
        for k in range(e2e_steps):
            assert np.array_equal(seq_u[k].numpy(), ref_u), "e2e result differs"
    if dist is not None:
        tt = torch.tensor([e2e_ms], device=red_dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = tt.item()

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    # ---- roofline of the fused stage (SURVEY 8(d) algorithmic work); small
    # grids run it as the split kernel + its ordered reduction (2 launches)
    stage_kernels = int(round(launches / (args.steps * cfg.T)))
    # batch fork (tnrd_despeckle, DESIGN.md 7b item 5): the half batch still
    # has >= 3 waves of 64x64 tiles at 2 CTAs per SM -> two tile-kernel
    # launches per stage, one per half, on two streams
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    half_tiles = -(-H // 64) * -(-W // 64) * (px_rank // (H * W) // 2)
    forked = (cfg.name != "c4" and px_rank > H * W and half_tiles >= 3 * 2 * sms
              and os.environ.get("TNRD_BATCH_FORK", "1")[:1] != "0")
    if forked and stage_kernels == 2:
        stage_kernels = "stage_kernel (fused tile kernel) x 2 batch halves on two streams"
    else:
        stage_kernels = {1: "stage_kernel (fused tile kernel)",
                         2: "stage_kernel_split + stage_reduce_kernel"}.get(stage_kernels, str(stage_kernels))
    px_launch = px_rank
    flop_launch = w_flop(cfg) * px_launch
    achieved_tf = flop_launch / (launch_ms * 1e-3) / 1e12
    peak_tf = peaks["fp32_tflops"]
    peak_sfu = peaks["mufu_ex2_gops"] * 1e9
    t_roof = max(w_flop(cfg) / (peak_tf * 1e12), w_sfu(cfg) / peak_sfu)  # s per pixel-stage
    roof_pxst = 1.0 / t_roof / 1e6                                        # MPix*stages/s
    ach_pxst = px_launch / (launch_ms * 1e-3) / 1e6
    traffic = None
    tpath = os.path.join(REPO, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(cfg.name)
    # what the stage kernel executes (ncu --set full SASS counts, committed
    # under profiles/) at this run's live launch time: the executed FP32
    # rate, which -- unlike SURVEY's algorithmic count -- cannot exceed peak
    executed = None
    epath = os.path.join(REPO, "profiles", "executed.json")
    if os.path.exists(epath):
        ex = json.load(open(epath)).get(cfg.name)
        if ex:
            ex_tf = 2.0 * ex["ffma_per_px_stage"] * px_launch / (launch_ms * 1e-3) / 1e12
            executed = dict(ex, achieved_tflops=ex_tf, frac=ex_tf / peak_tf)
    conf = workload_config(cfg, args, B)
    if cfg.name == "c4":
        conf.update({"parallelism": f"row strips x{world}, {cfg.m - 1}-row u halo exchanged per stage (NCCL P2P)",
                     "rows_per_rank": px_rank // W})
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak" if cfg.batch == 1 and cfg.name != "c4" else "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": conf,
        "roofline": {
            "bound": "fp32", "unit": "TFLOP/s", "achieved": achieved_tf,
            "peak": peak_tf, "frac": achieved_tf / peak_tf, "traffic": traffic,
            "peak_source": "measured on this GPU by tnrd_probe (FFMA); MEASURED_PEAKS.json has no FP32/MUFU entry",
            "work": f"SURVEY 8(d): W_flop={w_flop(cfg)} FLOP/pixel-stage x {px_launch} px per stage",
            "launch_ms": launch_ms,
            "stage_kernels": stage_kernels,
            "executed": executed,
            "survey_combined": {
                "unit": "MPix*stages/s", "achieved": ach_pxst, "peak": roof_pxst,
                "frac": ach_pxst / roof_pxst,
                "rule": "t_roof = max(W_flop/P_fp32, W_sfu/P_mufu) with on-box P_fp32, P_mufu",
                "p_mufu_gops": peaks["mufu_ex2_gops"]},
        },
        "e2e": {"value": total_px / (e2e_ms * 1e3), "unit": UNIT,
                "h2d_bytes_per_step": int(f_host.nbytes),
                "d2h_bytes_per_step": int(f_host.nbytes) + 8,
                "path": e2e_path},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if SHARED_GPU:
        line["not_a_measurement"] = (f"TNRD_BENCH_SHARED_GPU: {world} ranks shared cuda:0 "
                                     "(functional check of the N>1 path)")
    if world == 1 and not args.no_cpu_baseline:
        img0 = f_host[0] if cfg.name != "c4" else f_host[0][:512, :512]
        rate, dt, sample, threads = cpu_reference_run(cfg, model, img0, 20.0)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": threads,
                                "kind": "port", "sample": sample, **host_info(),
                                "single_core": single_core_run(cfg, model, img0)}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
