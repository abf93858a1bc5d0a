"""Strip sharding host logic (paper_1408_3526_b200/strips.py) on CPU:
the plan's bookkeeping, and the per-frame halo exchange on a real
world_size-2 gloo process group (127.0.0.1)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1408_3526_b200 import default_params
from paper_1408_3526_b200.strips import exchange_halo, plan_strips


def test_plan_covers_every_row_once(params):
    for h, world in ((512, 2), (512, 8), (4096, 8), (130, 3)):
        plans = plan_strips(params, h, world)
        assert plans[0].a0 == 0 and plans[-1].a1 == h
        for a, b in zip(plans, plans[1:]):
            assert a.a1 == b.a0
            assert b.halo == params.my - 1 and b.lo == b.a0 - 8
        assert plans[0].halo == 0
        assert max(p.a1 - p.a0 for p in plans) - min(p.a1 - p.a0 for p in plans) <= 1


def test_plan_rejects_thin_strips(params):
    with pytest.raises(ValueError):
        plan_strips(params, 40, 8)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, height, width, result):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = default_params()
    plan = plan_strips(p, height, world)[rank]
    full = torch.arange(height * width, dtype=torch.float32).reshape(height, width)
    ok = True
    for frame in range(3):
        g = full + 1000.0 * frame
        own = g[plan.a0:plan.a1].clone()
        halo = exchange_halo(own, plan, p.my - 1)
        local = own if halo is None else torch.cat([halo, own])
        ok &= bool(torch.equal(local, g[plan.lo:plan.a1]))
    result[rank] = int(ok)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_halo_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    result = ctx.Array("i", [0] * world)
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 64, 20, result)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    assert list(result) == [1] * world
