"""Row-strip sharding of one large scene across ranks (BASELINE config C4).

Each rank owns rows [row0, row1) of the scene plus h = 2r = m - 1 halo rows
on every internal edge.  Before every stage the current u's h boundary rows
are exchanged with the strip neighbours (torch.distributed P2P: NCCL over
NVLink on GPUs, gloo on CPU for the tests); the fused stage kernel then runs
on the strip with TNRD_STAGE_TOP_HALO / BOTTOM_HALO so that only the true
image top/bottom are mirrored.

Why h = m - 1 rows of u (not r): one stage needs phi on an r-row band
around the strip, and phi there needs u another r rows further out
(a 3-row halo gives max abs error 0.33, 6 rows gives 0).
The kernel consumes u rows -2r..-1 directly, so one exchange of u per stage
is enough and no phi crosses the link.

The stage operator is pluggable (``stage_fn``) so the partitioning and
exchange logic is tested on CPU with the float64 oracle as the operator
(tests/test_strips_cpu.py) and on the GPU with the fused kernel.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

from . import _lib


def strip_bounds(H: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced row ranges (first H % world strips get +1)."""
    base, extra = divmod(H, world)
    row0 = rank * base + min(rank, extra)
    return row0, row0 + base + (1 if rank < extra else 0)


@dataclass
class StripLayout:
    H: int
    W: int
    world: int
    rank: int
    halo: int  # rows of u exchanged per internal edge (= m - 1)

    @property
    def rows(self) -> tuple[int, int]:
        return strip_bounds(self.H, self.world, self.rank)

    @property
    def n(self) -> int:
        r0, r1 = self.rows
        return r1 - r0

    @property
    def has_top(self) -> bool:
        return self.rank > 0

    @property
    def has_bottom(self) -> bool:
        return self.rank < self.world - 1

    @property
    def flags(self) -> int:
        return ((_lib.STAGE_TOP_HALO if self.has_top else 0) |
                (_lib.STAGE_BOTTOM_HALO if self.has_bottom else 0))

    def check(self) -> None:
        if self.world > 1 and self.n < self.halo:
            raise ValueError(f"strip of {self.n} rows is thinner than the "
                             f"{self.halo}-row halo; use fewer ranks")


def exchange_halos(buf, layout: StripLayout, group=None) -> None:
    """Fill the halo rows of ``buf`` ((n + 2h) x W, strip rows at [h, h+n))
    from the neighbours: my first h rows go up, my last h rows go down."""
    import torch.distributed as dist
    h, n = layout.halo, layout.n
    ops = []
    if layout.has_top:
        up = layout.rank - 1
        ops.append(dist.P2POp(dist.isend, buf[h:2 * h].contiguous(), up, group))
        ops.append(dist.P2POp(dist.irecv, buf[0:h], up, group))
    if layout.has_bottom:
        down = layout.rank + 1
        ops.append(dist.P2POp(dist.isend, buf[n:n + h].contiguous(), down, group))
        ops.append(dist.P2POp(dist.irecv, buf[n + h:n + 2 * h], down, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


def exchange_halos_host(buf, layout: StripLayout, group=None) -> None:
    """exchange_halos through host memory: the boundary rows are copied to
    CPU tensors, exchanged with a CPU backend (gloo) and copied back.  For
    process groups without device P2P (gloo, or several ranks sharing one
    GPU in bench.py's TNRD_BENCH_SHARED_GPU functional check)."""
    import torch.distributed as dist
    h, n = layout.halo, layout.n
    ops, back = [], []
    if layout.has_top:
        up = layout.rank - 1
        ops.append(dist.P2POp(dist.isend, buf[h:2 * h].cpu(), up, group))
        rt = buf.new_empty((h,) + tuple(buf.shape[1:]), device="cpu")
        ops.append(dist.P2POp(dist.irecv, rt, up, group))
        back.append((slice(0, h), rt))
    if layout.has_bottom:
        down = layout.rank + 1
        ops.append(dist.P2POp(dist.isend, buf[n:n + h].cpu(), down, group))
        rb = buf.new_empty((h,) + tuple(buf.shape[1:]), device="cpu")
        ops.append(dist.P2POp(dist.irecv, rb, down, group))
        back.append((slice(n + h, n + 2 * h), rb))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for sl, t in back:
        buf[sl].copy_(t)


StageFn = Callable[[int, object, object, object, StripLayout, int], None]


def run_strip(f_ext, stage_fn: StageFn, T: int, layout: StripLayout,
              bufs, exchange=exchange_halos, group=None):
    """Despeckle one strip.  ``f_ext`` holds the strip's f at rows [h, h+n)
    (its halo rows are filled here); ``bufs`` are two scratch tensors shaped
    like f_ext.  ``stage_fn(t, u_in, f, u_out, layout, flags)`` computes rows
    [h, h+n) of u_out.  Returns the buffer holding u_T (rows [h, h+n))."""
    layout.check()
    exchange(f_ext, layout, group)          # stage 0 reads u_0 = max(f, 1e-6)
    cur = f_ext
    for t in range(T):
        if t > 0:
            exchange(cur, layout, group)
        dst = bufs[t % 2]
        fl = layout.flags
        if t == 0:
            fl |= _lib.STAGE_FLOOR_INPUT | _lib.STAGE_CHECK_F
        stage_fn(t, cur, f_ext, dst, layout, fl)
        cur = dst
    return cur


def gpu_stage_fn(device_model, status=None, stream=None) -> StageFn:
    """Stage operator = the fused sm_100a kernel on rows [h, h+n)."""
    def fn(t, u_in, f, u_out, layout, flags):
        device_model.stage(t, u_in, f, out=u_out, flags=flags, stream=stream,
                           status=status, rows=(layout.halo, layout.n))
    return fn
