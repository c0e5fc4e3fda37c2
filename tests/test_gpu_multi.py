"""N = 2 (or more) GPUs: the collective steps a3 (adv-norm allreduce), a8 (gradient allreduce +
Adam, over NCCL and over NVLink peer memory), a9 (preemption poll) and a10 (counts) through the C
ABI, one process per GPU.

Checks: parameters bit-identical on every rank after a learner step; the update
equals the oracle's N-rank learner step (per-tensor relative L2 of the parameter update, the
network tolerance); preemption lengths equal the oracle closed form bit-exactly; step
accounting is exact.  Skipped when fewer than 2 GPUs are visible."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        _worker_body(rank, world, port, q)
    except BaseException as e:  # report instead of leaving the parent waiting on the queue
        import traceback
        q.put((rank, {"error": traceback.format_exc()}))
        raise


def _worker_body(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    import paper_1911_00357_b200 as dd
    import synth
    from oracle import preempt
    from paper_1911_00357_b200.learner import Learner, preempt_collect
    obj = [dd.get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx = dd.Context(rank, world, obj[0], device=rank)
    obj2 = [dd.get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj2, src=0)
    out = {}
    # a10 before any learner is registered: the NCCL path
    out["counts_nccl"] = dd.ddppo_allreduce_counts(ctx, [rank + 5, 7]).tolist()
    # ---- learner step (gps, one rollout per rank, rank 1 preempted to 40 steps)
    c = synth.CONFIGS["gps"]
    desc = dd.model_desc("gps")
    lay = dd.param_layout(desc)
    P = dd.param_count(desc)
    p0 = synth.init_params([(off, int(np.prod(s)), fan) for _, off, s, fan in lay], P, 5)
    L = 128 if rank == 0 else 40
    ro = synth.rollout(c["E"], c["T"], 5, rank=rank, length=L)
    pm = synth.perms(5, 0, c["epochs"], c["E"], rank=rank)
    # S:L26 / S:L329: a layout disagreement at rendezvous is a protocol error on every rank
    try:
        dd.ddppo_layout_check(ctx, desc, c["E"] + rank, c["T"], 132, c["minibatches"], c["epochs"])
        out["protocol"] = None
    except dd.DdppoError as e:
        out["protocol"] = e.code
    # a8 over NCCL (unregistered workspace), then over NVLink peer memory (registered workspace; the
    # sharded reduce-scatter / Adam / all-gather form, then the all-read form on a second context)
    for key, peer, mode in (("params_nccl", False, "sharded"), ("params_allread", True, "allread"),
                            ("params", True, "sharded")):
        cx = ctx
        if key == "params_allread":  # one registered workspace per context
            cx = dd.Context(rank, world, obj2[0], device=rank)
        dd.ddppo_set_a8_mode(cx, mode)
        lrn = Learner(cx, "gps", c["E"], c["T"], c["epochs"], c["minibatches"], params=p0, peer=peer,
                      normalize_adv=True)
        lrn.load_rollout(ro, pm)
        lrn.step()
        torch.cuda.synchronize()
        cx.check()
        out[key] = lrn.params.cpu().numpy()
        if cx is not ctx:
            cx.close()
    out["stats"] = lrn.stats.cpu().numpy()
    # a second rollout through the peer path (gradient double buffer continues across calls)
    ro2 = synth.rollout(c["E"], c["T"], 6, rank=rank, length=L)
    lrn.load_rollout(ro2, synth.perms(6, 1, c["epochs"], c["E"], rank=rank))
    lrn.step()
    torch.cuda.synchronize()
    ctx.check()
    out["params2"] = lrn.params.cpu().numpy()
    # ---- the Depth agent (TMA convolutions, side-stream weight gradients) over the sharded a8
    cd = synth.CONFIGS["depth"]
    dsc = dd.model_desc("depth")
    Pd = dd.param_count(dsc)
    pd0 = synth.init_params([(off, int(np.prod(s_)), fan) for _, off, s_, fan in dd.param_layout(dsc)], Pd, 8)
    obj3 = [dd.get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj3, src=0)
    cxd = dd.Context(rank, world, obj3[0], device=rank)
    lrd = Learner(cxd, "depth", cd["E"], 16, cd["epochs"], cd["minibatches"], params=pd0, normalize_adv=True)
    for it in range(3):
        lrd.load_rollout(synth.rollout(cd["E"], 16, 8, rank=rank, iteration=it, length=16 if rank == 0 else 9,
                                       obs_shape=cd["obs"]), synth.perms(8, it, cd["epochs"], cd["E"], rank=rank))
        lrd.step()
    torch.cuda.synchronize()
    cxd.check()
    out["depth_params"] = lrd.params.cpu().numpy()
    out["depth_moved"] = float(np.abs(out["depth_params"] - pd0).max())
    cxd.close()
    # ---- NEXT-1: collection by the policy itself under the preemption protocol in wall-clock ticks
    # (the poll runs over the registered learner's NVLink peer areas), then the learner step
    from paper_1911_00357_b200.collect import Collector
    Tc = 24
    costs_c = synth.straggler_costs(11, world, Tc, lo=1.0, hi=6.0)
    costs_c[world - 1] *= 4
    lrc = Learner(ctx, "gps", c["E"], Tc, c["epochs"], c["minibatches"], params=p0, peer=False, normalize_adv=True)
    col = Collector(lrc, synth.PointGoalEnv(c["E"], 12, rank=rank), seed=12 + rank)
    roc = col.collect(Tc, costs=costs_c[rank], p_percent=50, tick_s=1e-4)
    out["L_collect"] = int(roc["length"][0])
    out["L_collect_ref"] = int(preempt.closed_form_lengths(costs_c, Tc, 50)[rank])
    lrc.load_rollout(roc, synth.perms(12, 0, c["epochs"], c["E"], rank=rank))
    lrc.step()
    torch.cuda.synchronize()
    ctx.check()
    out["collect_params"] = lrc.params.cpu().numpy()
    # ---- a10 counts
    out["counts"] = dd.ddppo_allreduce_counts(ctx, [c["E"] * L, rank + 1]).tolist()
    # (registered learner: the NVLink exchange; repeated calls cycle its double-buffered slots)
    out["counts_rep"] = [dd.ddppo_allreduce_counts(ctx, [10 * i + rank, -i]).tolist() for i in range(5)]
    # ---- a9 preemption over NCCL (virtual ticks)
    T = 32
    costs = synth.straggler_costs(7, world, T, lo=1.0, hi=8.0)
    costs[world - 1] *= 5
    out["L"], out["ticks"] = preempt_collect(ctx, costs[rank], T, 60)
    out["L_ref"] = preempt.closed_form_lengths(costs, T, 60)[rank]
    q.put((rank, out))
    ctx.close()
    dist.destroy_process_group()


def test_two_rank_learner_step_and_protocols():
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    import torch.multiprocessing as mp

    import synth
    from oracle import learner

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for r in range(world):
        assert "error" not in res[r], res[r]["error"]
    for p in procs:
        p.join(timeout=120)
    for key in ("params", "params_nccl", "params2", "params_allread", "depth_params", "collect_params"):
        assert np.array_equal(res[0][key], res[1][key]), key  # rank-identical
    assert res[0]["protocol"] == res[1]["protocol"] == 3  # DDPPO_ERR_PROTOCOL on both ranks
    assert res[0]["depth_moved"] > 1e-4
    # the two peer a8 forms differ only in the association order of the clip norm's fp64 partials
    d = np.abs(res[0]["params"].astype(np.float64) - res[0]["params_allread"]).max()
    assert d < 1e-6, d
    # oracle: the same two rollouts in one process
    import paper_1911_00357_b200 as dd
    c = synth.CONFIGS["gps"]
    desc = dd.model_desc("gps")
    lay = dd.param_layout(desc)
    P = dd.param_count(desc)
    p0 = synth.init_params([(off, int(np.prod(s)), fan) for _, off, s, fan in lay], P, 5)
    ros = [synth.rollout(c["E"], c["T"], 5, rank=r, length=128 if r == 0 else 40) for r in range(world)]
    pms = [synth.perms(5, 0, c["epochs"], c["E"], rank=r) for r in range(world)]
    po, _, _, _, info = learner.learner_step("gps", p0, np.zeros(P), np.zeros(P), 0, ros, pms,
                                             dict(epochs=c["epochs"], minibatches=c["minibatches"]))
    dpo = po - p0
    for key in ("params", "params_nccl", "params_allread"):
        dp = res[0][key].astype(np.float64) - p0
        for name, off, shape, _ in lay:
            n = int(np.prod(shape))
            e = np.linalg.norm(dp[off:off + n] - dpo[off:off + n]) / np.linalg.norm(dpo[off:off + n])
            assert e < 5e-2, (key, name, e)
    assert res[0]["counts_nccl"] == res[1]["counts_nccl"] == [11, 14]
    assert res[0]["counts"] == res[1]["counts"] == [c["E"] * (128 + 40), 3]
    assert res[0]["counts_rep"] == res[1]["counts_rep"] == [[20 * i + 1, -2 * i] for i in range(5)]
    for r in range(world):
        assert res[r]["L"] == res[r]["L_ref"]
        assert res[r]["L_collect"] == res[r]["L_collect_ref"]
    assert res[0]["L_collect"] == 24 > res[1]["L_collect"]  # the slow rank was preempted
    assert res[0]["ticks"] == res[1]["ticks"]
