"""Device-resident buffers around ddppo_learner_step (one DD-PPO worker = one GPU).

Holds the rollout arrays in HBM (env-major [E][ld] rows, include/ddppo.h), the fp32 master
parameters and Adam moments, and the workspace; `step()` is one call into the C ABI.  The
preemption driver realises P:L171 with ddppo_preempt_poll (one int32 allreduce per tick).
"""
import ctypes

import numpy as np
import torch

from . import (Rollout, adam_cfg, ddppo_layout_check, ddppo_learner_register, ddppo_learner_step, ddppo_preempt_poll,
               learner_workspace_size, learner_cfg,
               loss_cfg, model_desc, param_count, param_layout, preempt_cfg, visual_obs)

ROLLOUT_FIELDS = {  # name -> torch dtype
    "rew": torch.float32, "val": torch.float32, "done": torch.uint8, "length": torch.int32,
    "goal": torch.float32, "prev_action": torch.int32, "mask": torch.float32, "h0": torch.float32,
    "action": torch.int32, "logp_old": torch.float32, "obs": torch.bfloat16, "c0": torch.float32,
    "obs_rgb": torch.uint8,
}
# depth frames (bf16) of the Depth (configs[2]) / RGB-D (configs[3]) agents; RGB-D camera bytes
OBS_SHAPES = {2: (1, 64, 64), 3: (1, 256, 256), 4: (1, 256, 256), 5: (1, 256, 256)}
RGB_SHAPE = (3, 256, 256)


class Learner:
    """normalize_adv defaults to the paper's setting (off); north_star's hot path (bench.py)
    turns it on explicitly."""
    def __init__(self, ctx, arch, E, T, epochs=2, minibatches=2, hidden=None, params=None, device="cuda",
                 normalize_adv=False, use_value_clip=True, lr=2.5e-4, max_grad_norm=0.5, ld=None, adam_eps=1e-8,
                 peer=True, freeze_encoder=False, freeze_mask=None, rollout_buffers=1):
        self.ctx, self.E, self.T = ctx, E, T
        self.ld = ld or ((T + 1 + 3) // 4 * 4)
        self.epochs, self.minibatches = epochs, minibatches
        self.desc = model_desc(arch, hidden)
        self.hidden = self.desc.hidden
        self.P = param_count(self.desc)
        self.layout = param_layout(self.desc)
        dev = torch.device(device)
        self.device = dev
        f32 = dict(dtype=torch.float32, device=dev)
        self.params = torch.zeros(self.P, **f32) if params is None else torch.as_tensor(params, **f32).clone()
        self.m = torch.zeros(self.P, **f32)
        self.v = torch.zeros(self.P, **f32)
        self.adam_step = 0
        self.cfg = learner_cfg(epochs, minibatches, normalize_adv=normalize_adv,
                               loss=loss_cfg(use_value_clip=use_value_clip, normalize_adv=normalize_adv),
                               adam=adam_cfg(0, lr=lr, eps=adam_eps, max_grad_norm=max_grad_norm))
        # transfer mechanics (NEXT-4): a frozen visual encoder and / or a per-entry freeze mask
        self.cfg.freeze_encoder = int(freeze_encoder)
        self.freeze_mask = None
        if freeze_mask is not None:
            self.freeze_mask = torch.as_tensor(np.asarray(freeze_mask, dtype=np.uint8)).to(dev).contiguous()
            self.cfg.freeze_mask = self.freeze_mask.data_ptr()
        wsb = learner_workspace_size(self.desc, E, T, self.ld, minibatches, epochs)
        self.ws = torch.empty(wsb // 4 + 64, **f32)
        if getattr(ctx, "world", 1) > 1:
            ddppo_layout_check(ctx, self.desc, E, T, self.ld, minibatches, epochs)  # S:L26 (collective)
            if peer:
                ddppo_learner_register(ctx, self.ws)  # a8 over NVLink peer memory (collective)
        ld = self.ld
        self.rnn_layers = 2 if self.desc.arch in (3, 4, 5) else 1  # the RGB-D agents: 2 LSTM layers
        hs = self.rnn_layers * self.hidden
        shapes = {"rew": (E, ld), "val": (E, ld), "done": (E, ld), "length": (E,), "goal": (E, T, 3),
                  "prev_action": (E, ld), "mask": (E, ld), "h0": (E, hs), "action": (E, ld),
                  "logp_old": (E, ld)}
        if self.desc.arch in (2, 3, 4, 5):  # visual agents: + frames and the LSTM cell state
            shapes.update(obs=(E, T) + OBS_SHAPES[self.desc.arch], c0=(E, hs))
        if self.desc.arch in (3, 4, 5):
            shapes["obs_rgb"] = (E, T) + RGB_SHAPE
        # all rollout arrays + the epoch permutations in one device arena (256-byte aligned fields), so a
        # packed host arena reaches HBM in a single copy
        shapes["perms"] = (epochs, E)
        self._layout, off = {}, 0
        for k, shp in shapes.items():
            dt = ROLLOUT_FIELDS.get(k, torch.int32)
            nbytes = int(np.prod(shp)) * torch.empty((), dtype=dt).element_size()
            self._layout[k] = (off, shp, dt, nbytes)
            off = (off + nbytes + 255) // 256 * 256
        self._arena_bytes = off
        # rollout_buffers = 2: two device arenas, so the next rollout's H2D copy (load_rollout with a
        # copy stream) overlaps the current learner step; each arena is its own CUDA-graph key
        self.shapes_nop = [k for k in shapes if k != "perms"]
        self._arenas = [torch.zeros(off, dtype=torch.uint8, device=dev) for _ in range(max(1, rollout_buffers))]
        self._ready = [None] * len(self._arenas)   # copy-stream event: the arena holds its rollout
        self._free = [None] * len(self._arenas)    # step-stream event: the last step reading it is done
        self._next = 0                              # the arena load_rollout fills next
        self._use(0)
        self.adv = torch.zeros((E, ld), **f32)
        self.ret = torch.zeros((E, ld), **f32)
        self.stats = torch.zeros((epochs * minibatches, 8), **f32)
        self.host_len = np.full(E, T, np.int32)
        self.host_perms = np.zeros((epochs, E), np.int32)
        self.shapes = shapes

    # --------------------------------------------------------------- inputs
    def _use(self, i):
        self._cur = i
        self.arena = self._arenas[i]
        self.dev = {k: self._view(self.arena, k) for k in self.shapes_nop}
        self.perms = self._view(self.arena, "perms")

    def _view(self, arena, k):
        off, shp, dt, nbytes = self._layout[k]
        return arena[off:off + nbytes].view(dt).view(shp)

    def pinned_host_buffers(self):
        """Page-locked host mirror of the rollout arena (views per field, incl. "perms"); loading it is
        one H2D copy."""
        arena = torch.zeros(self._arena_bytes, dtype=torch.uint8).pin_memory()
        views = {k: self._view(arena, k) for k in self._layout}
        views["__arena__"] = arena
        return views

    def host_fields(self, ro):
        """A synth rollout dict -> {field: host array in the device arena's dtype} (float frames ->
        bf16 depth + uint8 RGB; dtype marshalling only)."""
        out = {k: ro[k] for k in self.dev if k not in ("obs", "obs_rgb")}
        if "obs" in self.dev:
            out.update(visual_obs(ro["obs"], self.desc.arch in (3, 4, 5)))
        return out

    def load_rollout(self, ro, perms, non_blocking=False, copy_stream=None):
        """Copy a rollout (synth dict of numpy arrays, or a pinned_host_buffers() arena) + perms to HBM.
        With rollout_buffers = 2 and a packed arena, `copy_stream` carries the H2D copy into the arena
        the next step() will read, after the step that last read that arena."""
        if "__arena__" in ro:  # packed pinned arena: perms are inside it
            ro["perms"].copy_(torch.as_tensor(np.asarray(perms, dtype=np.int32)))
            i = 0
            if copy_stream is not None:  # alternate the arenas only for stream-overlapped loads
                i = self._next
                self._next = (i + 1) % len(self._arenas)
            self._use(i)
            if copy_stream is not None:
                if self._free[i] is not None:
                    copy_stream.wait_event(self._free[i])
                with torch.cuda.stream(copy_stream):
                    self.arena.copy_(ro["__arena__"], non_blocking=non_blocking)
                    self._ready[i] = torch.cuda.Event()
                    self._ready[i].record(copy_stream)
            else:
                self.arena.copy_(ro["__arena__"], non_blocking=non_blocking)
                self._ready[i] = None
            self.host_perms[:] = ro["perms"].numpy()
            self.host_len[:] = ro["length"].numpy()
            return
        ro = self.host_fields(ro) if "obs" in self.dev and ro["obs"].dtype != torch.bfloat16 else ro
        for k in self.dev:
            src = ro[k]
            if isinstance(src, np.ndarray):
                src = torch.from_numpy(np.ascontiguousarray(src))
            self.dev[k].copy_(src.reshape(self.dev[k].shape), non_blocking=non_blocking)
        p = perms if isinstance(perms, np.ndarray) else perms.numpy()
        self.host_perms[:] = p
        self.perms.copy_(torch.from_numpy(np.ascontiguousarray(self.host_perms)), non_blocking=non_blocking)
        lens = ro["length"]
        self.host_len[:] = lens.numpy() if isinstance(lens, torch.Tensor) else lens

    # --------------------------------------------------------------- the learner step
    def _rollout_struct(self):
        r = Rollout()
        d = self.dev
        r.rew, r.val, r.done, r.len = d["rew"].data_ptr(), d["val"].data_ptr(), d["done"].data_ptr(), \
            d["length"].data_ptr()
        r.goal, r.prev_action, r.mask, r.h0 = d["goal"].data_ptr(), d["prev_action"].data_ptr(), \
            d["mask"].data_ptr(), d["h0"].data_ptr()
        r.action, r.logp_old, r.perms = d["action"].data_ptr(), d["logp_old"].data_ptr(), self.perms.data_ptr()
        r.host_len = self.host_len.ctypes.data
        r.host_perms = self.host_perms.ctypes.data
        r.E, r.T, r.ld = self.E, self.T, self.ld
        if "obs" in d:
            r.obs, r.c0 = d["obs"].data_ptr(), d["c0"].data_ptr()
        if "obs_rgb" in d:
            r.obs_rgb = d["obs_rgb"].data_ptr()
        return r

    def step(self, stream=None, stats=None):
        """One learner step (stream-ordered).  `stats` (optional [epochs*minibatches][8] CUDA tensor)
        receives the loss statistics instead of self.stats (double-buffering for pipelined reads)."""
        self.cfg.adam.step = self.adam_step
        i = self._cur
        st = stream if stream is not None else torch.cuda.current_stream()
        if self._ready[i] is not None:  # the arena's H2D copy ran on a copy stream
            st.wait_event(self._ready[i])
            self._ready[i] = None
        self._ro = self._rollout_struct()
        out = self.stats if stats is None else stats
        self.adam_step = ddppo_learner_step(self.ctx, self.desc, self._ro, self.cfg, self.params, self.m, self.v,
                                            self.adv, self.ret, out, self.ws, stream)
        if len(self._arenas) > 1:
            self._free[i] = torch.cuda.Event()
            self._free[i].record(st)
        return out

    def steps_per_rollout(self):
        """The a10 input of this rank (ddppo_rollout_steps: sum_e min(len_e, T))."""
        from . import ddppo_rollout_steps
        return ddppo_rollout_steps(self.host_len, self.T)


def preempt_collect(ctx, step_costs, T, p_percent, exchange=None, world=None, on_step=None,
                    other_workers=False, tick_s=0.0):
    """Collection phase of one rank under the preemption protocol, in virtual ticks.

    step_costs: this rank's per-step costs in ticks (>= 1).  Every tick an active rank advances
    its current step; then all ranks exchange {finished, active} -- ddppo_preempt_poll, one int32
    allreduce standing in for the paper's TCPStore counter -- and a rank that
    just completed a step applies the threshold decision (computed by the C library).  Ranks
    that stopped keep polling; everybody leaves on the first tick whose exchange shows no
    active rank.  `exchange(finished, active) -> (finished_count, active_count)` replaces the
    NCCL poll in the gloo CPU tests (then `world` must be given).  tick_s > 0: wall-clock mode (SURVEY
    8 c-9) -- every tick lasts at least tick_s seconds of real time (the work of a completed step,
    on_step, runs inside its tick); the decisions stay exact because each tick's exchange is
    synchronous.  Returns (L, ticks).
    """
    import time
    from . import ddppo_preempt_decide
    cfg = preempt_cfg(p_percent, T, other_workers=other_workers)
    if world is None:
        world = ctx.world
    steps, elapsed, tick, active, finished = 0, 0, 0, True, False
    t_next = time.perf_counter()
    while True:
        tick += 1
        just = False
        if tick_s > 0:
            t_next += tick_s
            while time.perf_counter() < t_next:
                pass
        if active:
            elapsed += 1
            if elapsed == int(step_costs[steps]):
                steps += 1
                elapsed = 0
                just = True
                finished = steps == T
                if on_step is not None:
                    on_step(steps)
        if exchange is None:
            stop, fin, act = ddppo_preempt_poll(ctx, steps, finished, active, cfg)
        else:
            fin, act = exchange(int(finished), int(active))
            stop = ddppo_preempt_decide(cfg, world, steps, fin)
        if act == 0:
            return steps, tick
        if just and active and stop:
            active = False


def reinit_critic(lrn, seed):
    """P:L405 "critic layers are reinitialized" on a Learner's parameters (and their Adam moments)."""
    from . import ddppo_reinit_critic
    ddppo_reinit_critic(lrn.ctx, lrn.desc, lrn.params, lrn.m, lrn.v, seed)
