"""Spatial strip sharding of one frame stream across GPUs.

Anchor (y, x) of frame n depends on input rows y-My+1 .. y of frames
n-Mz+1 .. n and on its own per-pixel state only (_kernels.py:31-90,
SPEC.md:150), plus I(n - mhat_z) at anchor - mhat.  So a frame splits
into horizontal strips of anchor rows, one per rank, and the only
exchange per frame is one-sided: rank g needs the My-1 input rows just
above its strip, which rank g-1 owns.  There is no reduction.

Each rank runs an ordinary device Pipeline on its local strip
[a0 - halo, a1) with ``halo_rows = My - 1`` input-only rows on top
(cw_create(..., halo_rows, row_offset)); the halo is a point-to-point
send/recv over torch.distributed (NCCL over NVLink on a GPU box, gloo in
the CPU tests) of My-1 rows, 8 x W x 4 bytes per frame.

Outputs: the residual of local anchor rows [halo, H_local) lands at global
output rows [a0 - mhat_y, a1 - mhat_y) (pipeline.py:41-50 geometry), and
the velocity field covers global anchor rows [a0, a1).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .params import FilterParams, validate

__all__ = ["StripPlan", "plan_strips", "exchange_halo", "StripPipeline"]


@dataclass(frozen=True)
class StripPlan:
    """Rows owned by one rank.

    a0, a1   : global anchor rows [a0, a1) this rank produces
    halo     : input-only rows received from rank - 1 (0 on rank 0)
    lo       : global row of local row 0 (= a0 - halo)
    """

    rank: int
    world: int
    a0: int
    a1: int
    halo: int

    @property
    def lo(self) -> int:
        return self.a0 - self.halo

    @property
    def local_height(self) -> int:
        return self.a1 - self.lo


def plan_strips(params: FilterParams, height: int, world: int) -> list[StripPlan]:
    """Equal strips of anchor rows (the remainder goes to the first ranks).
    Every rank but the first receives My-1 halo rows; every strip must hold
    at least My-1 rows so that the halo comes from a single neighbour."""
    validate(params)
    halo = params.my - 1
    if world < 1:
        raise ValueError("world size must be >= 1")
    base, extra = divmod(height, world)
    plans, a0 = [], 0
    for g in range(world):
        rows = base + (1 if g < extra else 0)
        a1 = a0 + rows
        plans.append(StripPlan(rank=g, world=world, a0=a0, a1=a1, halo=0 if g == 0 else halo))
        a0 = a1
    if world > 1 and min(p.a1 - p.a0 for p in plans) < halo:
        raise ValueError(f"strips of {base} rows are thinner than the {halo}-row halo")
    if plans[0].a1 - plans[0].a0 < params.my:
        raise ValueError("the first strip must hold a full analysis window")
    return plans


def exchange_halo(own_rows, plan: StripPlan, halo: int, group=None):
    """Send this rank's last ``halo`` rows to rank+1 and receive rank-1's
    (returned; None on rank 0).  ``own_rows`` is the (a1 - a0, W) torch
    tensor of this rank's rows (CUDA with NCCL, CPU with gloo).  One
    batched isend/irecv pair per neighbour, no collective."""
    import torch
    import torch.distributed as dist

    if plan.world == 1:
        return None  # one strip: nothing crosses
    # gloo moves host tensors only: stage CUDA rows through the host there
    staged = own_rows.is_cuda and dist.get_backend(group) == "gloo"
    dev = own_rows.device
    ops, recv = [], None
    if plan.halo:
        recv = torch.empty((plan.halo, own_rows.shape[1]), dtype=own_rows.dtype,
                           device="cpu" if staged else dev)
        ops.append(dist.P2POp(dist.irecv, recv, plan.rank - 1, group=group))
    if plan.rank + 1 < plan.world:
        send = own_rows[-halo:].contiguous()
        ops.append(dist.P2POp(dist.isend, send.cpu() if staged else send, plan.rank + 1, group=group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    if staged and recv is not None:
        recv = recv.to(dev)
    return recv


class StripPipeline:
    """One rank's share of a strip-sharded stream (device Pipeline + halo).

    ``process_frame(own_rows)`` takes this rank's (a1 - a0, W) rows as a
    CUDA tensor, receives the halo, runs the fused kernel on the local strip
    and returns the local WhitenedOutput (None during warm-up) together
    with the global row offsets of its residual and velocity arrays.
    """

    def __init__(self, params: FilterParams, width: int, height: int, rank: int, world: int,
                 group=None, device: int = 0, bank=None):
        import torch

        from .pipeline import Pipeline

        self.params = params
        self.plans = plan_strips(params, height, world)
        self.plan = self.plans[rank]
        self.halo = params.my - 1
        self.group = group
        self.width = width
        self.device = torch.device("cuda", device)
        self.pipe = Pipeline(params, width, self.plan.local_height, device=device, bank=bank,
                             _strip=(self.plan.halo, self.plan.lo))
        # two assembly buffers: frame n+1 is assembled while frame n's copy
        # into the pipeline's ring slot may still be queued
        self._frames = [torch.empty((self.plan.local_height, width), dtype=torch.float32, device=self.device)
                        for _ in range(2)]
        self._k = 0

    def assemble(self, own_rows):
        """Local strip frame = [halo rows from rank-1 ; own rows], on torch's
        current stream."""
        frame = self._frames[self._k & 1]
        self._k += 1
        halo = exchange_halo(own_rows, self.plan, self.halo, self.group)
        if halo is not None:
            frame[: self.plan.halo].copy_(halo)
        frame[self.plan.halo:].copy_(own_rows)
        return frame

    def process_frame(self, own_rows):
        return self.pipe.process_frame_device(self.assemble(own_rows))

    def process_stream(self, rows, depth: int = 3):
        """Pipelined ``process_frame`` over an iterable of this rank's
        (a1 - a0, W) CUDA row blocks: the halo exchange and assembly of frame
        n+1, the fused kernel of frame n and the download of frame n-1 into
        pinned host buffers overlap (cw_submit_device / cw_wait).  Yields the
        local WhitenedOutput of every ready frame, in order."""
        import ctypes
        from collections import deque

        import torch

        from . import _native

        lib = _native.load()
        pipe = self.pipe
        h, w = self.plan.local_height, self.width
        inflight: deque = deque()

        def collect():
            ticket, res, pred, vidx = inflight.popleft()
            ready, fidx = ctypes.c_int32(0), ctypes.c_int64(-1)
            _native.check(lib.cw_wait(pipe._h, ticket, ctypes.byref(ready), ctypes.byref(fidx)), pipe._h)
            return pipe._wrap(int(fidx.value), res, pred, vidx, ticket=ticket) if ready.value else None

        try:
            for own in rows:
                frame = self.assemble(own)
                res, pred, vidx = pipe._pool.take_outputs(h, w, pipe._idx_bytes)
                ticket = ctypes.c_int64(-1)
                stream = torch.cuda.current_stream(self.device)
                _native.check(lib.cw_submit_device(pipe._h, ctypes.c_void_p(frame.data_ptr()), res.ctypes.data,
                                                   pred.ctypes.data, vidx.ctypes.data, ctypes.byref(ticket),
                                                   ctypes.c_void_p(stream.cuda_stream)), pipe._h)
                inflight.append((ticket.value, res, pred, vidx))
                while len(inflight) > depth:
                    out = collect()
                    if out is not None:
                        yield out
            while inflight:
                out = collect()
                if out is not None:
                    yield out
        finally:
            while inflight:
                lib.cw_wait(pipe._h, inflight.popleft()[0], None, None)

    def output_rows(self):
        """(global first residual row, local slice) and (global first
        velocity row, local slice) of this rank's outputs."""
        mhy = self.params.mhat[1]
        p = self.plan
        res_local = slice(p.halo - mhy if p.halo else 0, p.local_height - mhy)
        res_global0 = p.lo + res_local.start
        vel_local = slice(p.halo, p.local_height)
        return (res_global0, res_local), (p.a0, vel_local)

    def close(self):
        self.pipe.close()
