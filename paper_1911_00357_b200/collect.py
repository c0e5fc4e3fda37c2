"""The collection side of a DD-PPO worker (NEXT-1): batched single-step inference over the GPU's
environments (ddppo_policy_act), the preemption threshold protocol during
collection (ddppo_preempt_poll per tick; straggler step costs in virtual or wall-clock
ticks), the bootstrap value, then the learner step -- and the benchmark procedure of P:L628 (10
collect + optimise cycles, the steps of the last 5 over their time).

Host-side driver only (argument marshalling, the synthetic environment's stepping, buffer
management): every policy evaluation runs in the library's kernels.
"""
import time

import numpy as np
import torch

from . import (act_workspace_size, ddppo_allreduce_counts, ddppo_policy_act, make_act_batch, visual_obs)
from .learner import preempt_collect


class Collector:
    """One worker's E environments stepped by the learner's current policy."""

    def __init__(self, lrn, env, seed=0):
        self.lrn, self.env, self.seed = lrn, env, seed
        self.ctx, self.desc = lrn.ctx, lrn.desc
        E, dev = lrn.E, lrn.device
        self.E = E
        self.visual = lrn.desc.arch in (2, 3, 4, 5)
        self.rgbd = lrn.desc.arch in (3, 4, 5)
        hs = lrn.rnn_layers * lrn.hidden
        f32 = dict(dtype=torch.float32, device=dev)
        # one-step staging arena in the rollout layout (T = 1, ld = 2): the act call's inputs
        self.goal = torch.zeros((E, 1, 3), **f32)
        self.prev = torch.zeros((E, 2), dtype=torch.int32, device=dev)
        self.mask = torch.zeros((E, 2), **f32)
        if self.visual:
            Hs = 256 if self.rgbd else 64
            self.obs = torch.zeros((E, 1, 1, Hs, Hs), dtype=torch.bfloat16, device=dev)
            self.obs_rgb = torch.zeros((E, 1, 3, Hs, Hs), dtype=torch.uint8, device=dev) if self.rgbd else None
        else:
            self.obs = self.obs_rgb = None
        self.h = [torch.zeros((E, hs), **f32) for _ in range(3)]  # current, next, scratch (bootstrap)
        self.c = [torch.zeros((E, hs), **f32) for _ in range(3)]
        self.actions = torch.zeros(E, dtype=torch.int32, device=dev)
        self.logp = torch.zeros(E, **f32)
        self.values = torch.zeros(E, **f32)
        self.host = {k: torch.zeros(E, dtype=t).pin_memory() for k, t in
                     (("actions", torch.int32), ("logp", torch.float32), ("values", torch.float32))}
        self.ws = torch.empty(act_workspace_size(self.desc, E) // 4 + 64, **f32)
        self.counter = 0
        self.stream = torch.cuda.current_stream()

    def _act(self, h_out, c_out):
        g, p, m, frames = self.env.observe()
        self.goal.copy_(torch.from_numpy(g).view(self.E, 1, 3), non_blocking=True)
        self.prev[:, 0].copy_(torch.from_numpy(p), non_blocking=True)
        self.mask[:, 0].copy_(torch.from_numpy(m), non_blocking=True)
        if self.visual:
            vo = visual_obs(frames[:, None], self.rgbd)
            self.obs.copy_(vo["obs"].view(self.obs.shape), non_blocking=True)
            if self.rgbd:
                self.obs_rgb.copy_(vo["obs_rgb"].view(self.obs_rgb.shape), non_blocking=True)
        ab = make_act_batch(self.goal, self.prev, self.mask, self.h[0], h_out, self.E, 1, 2, 0, self.seed,
                            self.counter, obs=self.obs, obs_rgb=self.obs_rgb,
                            c_in=self.c[0] if self.visual else None, c_out=c_out if self.visual else None)
        self.counter += 1
        ddppo_policy_act(self.ctx, self.desc, self.lrn.params, ab, self.actions, self.logp, self.values, self.ws)
        for k in self.host:
            self.host[k].copy_(getattr(self, k), non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return g, p, m, frames

    def _step(self, t):
        g, p, m, frames = self._act(self.h[1], self.c[1])
        a = self.host["actions"].numpy().copy()
        r, d = self.env.step(a)
        ro = self.ro
        ro["goal"][:, t] = g
        ro["prev_action"][:, t] = p
        ro["mask"][:, t] = m
        ro["action"][:, t] = a
        ro["logp_old"][:, t] = self.host["logp"].numpy()
        ro["val"][:, t] = self.host["values"].numpy()
        ro["rew"][:, t] = r
        ro["done"][:, t] = d
        if self.visual:
            ro["obs"][:, t] = frames
        self.h[0], self.h[1] = self.h[1], self.h[0]
        self.c[0], self.c[1] = self.c[1], self.c[0]

    def collect(self, T, costs=None, p_percent=100, tick_s=0.0):
        """One rollout of up to T steps (all envs of this worker stop together: the worker is the unit
        the preemption protocol preempts).  Returns the synth-style rollout dict (host)."""
        E, lrn = self.E, self.lrn
        ld = lrn.ld
        hs = lrn.rnn_layers * lrn.hidden
        ro = {"rew": np.zeros((E, ld), np.float32), "val": np.zeros((E, ld), np.float32),
              "done": np.zeros((E, ld), np.uint8), "action": np.zeros((E, ld), np.int32),
              "prev_action": np.zeros((E, ld), np.int32), "mask": np.zeros((E, ld), np.float32),
              "logp_old": np.zeros((E, ld), np.float32), "goal": np.zeros((E, T, 3), np.float32),
              "h0": self.h[0].cpu().numpy().reshape(E, hs).copy(), "E": E, "T": T, "ld": ld}
        if self.visual:
            ro["obs"] = np.zeros((E, T, 4 if self.rgbd else 1) + ((256, 256) if self.rgbd else (64, 64)), np.float32)
            ro["c0"] = self.c[0].cpu().numpy().reshape(E, hs).copy()
        self.ro = ro
        if costs is None:
            for t in range(T):
                self._step(t)
            L, ticks = T, T
        else:
            L, ticks = preempt_collect(self.ctx, costs, T, p_percent, on_step=lambda s: self._step(s - 1),
                                       tick_s=tick_s)
        # the bootstrap value V(s_L) (slot L of the value row, Z6); its state update is discarded
        self._act(self.h[2], self.c[2])
        ro["val"][:, L] = self.host["values"].numpy()
        ro["length"] = np.full(E, L, np.int32)
        self.ticks = ticks
        return ro


def run_cycles(lrn, col, T, perms_fn, cycles=10, timed=5, costs_fn=None, p_percent=100, tick_s=0.0):
    """`cycles` collect + optimise cycles; throughput = experience steps of the last `timed`
    cycles (summed over ranks, a10) / their wall time (max over ranks through the same exchange).
    Returns (steps_per_s, per-cycle [(L, collected_all_ranks, t_collect, t_learn)])."""
    log = []
    t0 = None
    steps = 0
    for i in range(cycles):
        if i == cycles - timed:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
        ta = time.perf_counter()
        ro = col.collect(T, None if costs_fn is None else costs_fn(i), p_percent, tick_s)
        tb = time.perf_counter()
        lrn.load_rollout(ro, perms_fn(i))
        lrn.step()
        cnt = ddppo_allreduce_counts(lrn.ctx, [lrn.steps_per_rollout()])
        torch.cuda.synchronize()
        tc = time.perf_counter()
        log.append((int(ro["length"][0]), int(cnt[0]), tb - ta, tc - tb))
        if t0 is not None:
            steps += int(cnt[0])
    el = time.perf_counter() - t0
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():  # the slowest rank's time
        t = torch.tensor([el], dtype=torch.float64, device=lrn.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
    return steps / el, log
