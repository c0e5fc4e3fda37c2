"""World-size-2/4 gloo runs of the preemption driver on CPU (the N>1 host logic of step a9).

Each rank runs paper_1911_00357_b200.learner.preempt_collect with a gloo all_reduce as the
exchange and the C library's decision; the resulting per-rank lengths must equal the oracle's
closed form bit for bit, and the step accounting allreduce must match."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import preempt


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, costs, T, p, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1911_00357_b200.learner import preempt_collect

    def exchange(finished, active):
        t = torch.tensor([finished, active], dtype=torch.int32)
        dist.all_reduce(t)
        return int(t[0]), int(t[1])

    L, ticks = preempt_collect(None, costs[rank], T, p, exchange=exchange, world=world)
    acc = torch.tensor([16 * L, 16 * (T - L)], dtype=torch.int64)  # a10 step accounting (E = 16)
    dist.all_reduce(acc)
    q.put((rank, L, ticks, acc.tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,p,seed", [(2, 60, 0), (2, 100, 1), (4, 60, 2), (4, 50, 3)])
def test_gloo_preemption_matches_closed_form(world, p, seed):
    T = 24
    costs = synth.straggler_costs(seed, world, T, lo=1.0, hi=12.0)
    costs[world - 1] *= 6  # a straggler
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, costs, T, p, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
    L = np.array([r[1] for r in res])
    ref = preempt.closed_form_lengths(costs, T, p)
    assert np.array_equal(L, ref), (L, ref)
    col, pre = preempt.step_accounting(ref, 16, T)
    assert all(r[3] == [col, pre] for r in res)
    assert len({r[2] for r in res}) == 1  # every rank leaves on the same tick
