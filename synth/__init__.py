"""Seeded synthetic inputs shared by the oracle-side tests and the CUDA path.

This module holds NONE of the method's arithmetic (no GAE, loss, network or
optimizer math): it only draws rollouts shaped like PointGoal episodes,
initial parameters, epoch permutations and straggler step costs from
seeded NumPy Philox generators.  Both the oracle tests and the GPU path
consume exactly these arrays; nothing here is ever computed by either side.

Recipe:
  * episodes: start geodesic distance d0 ~ U(1, 20) m, goal bearing
    theta ~ U(-pi, pi); 4 actions stop / forward 0.25 m / left 10 deg /
    right 10 deg; a stochastic scripted behaviour policy (forward
    0.6, turn-towards-goal 0.28, turn-away 0.1, stop 0.02; stop 0.97 once
    d <= 0.2 m); forward fails (collision, no motion) with prob 0.1;
    episodes end on stop or after 500 steps.
  * rewards: -(d_new - d_old) - 0.01 per step plus terminal
    2.5 * SPL on success, SPL = d0 / max(d0, path length).
  * goal input [d, cos theta, sin theta]; prev_action = start
    token A (= 4) after an episode start; mask_t = 1 - done_{t-1}.
  * V_hat = 2.5 exp(-d/10) - 0.05 d + N(0, 0.1^2) (a stand-in critic, fp32);
    logp_old = log-probability of the taken action under the behaviour
    policy; h0 ~ N(0, 0.1^2).
  * per-step arrays are env-major [E][ld] with ld = round_up(T+1, 4); value
    row slot L holds the bootstrap V_hat(s_L); everything past L is zero.
"""
import numpy as np

NUM_ACTIONS = 4
START_TOKEN = NUM_ACTIONS

# BASELINE.json configs
CONFIGS = {
    "toy": dict(arch="toy", E=2, T=4, epochs=1, minibatches=1, hidden=64),
    "gps": dict(arch="gps", E=4, T=128, epochs=2, minibatches=2, hidden=512),
    "stress_gps": dict(arch="gps", E=16, T=128, epochs=2, minibatches=2, hidden=512),
    "depth": dict(arch="depth", E=4, T=128, epochs=2, minibatches=2, hidden=512, obs=(1, 64, 64)),
    # configs[4]: the Depth agent with 16 envs/GPU, collection under the preemption protocol with
    # synthetic stragglers (p = 60 %, minimum T/4); SURVEY 8 pins the depth model for it
    # configs[3]: the paper-shaped RGB-D agent (half-width ResNet50 + 2-layer LSTM-512)
    "rgbd": dict(arch="rgbd", E=4, T=128, epochs=2, minibatches=2, hidden=512, obs=(4, 256, 256), rnn_layers=2),
    # NEXT-3: the RGB-D agent with the half-width SE-ResNeXt50 encoder (reading R9)
    "serx50": dict(arch="serx50", E=4, T=128, epochs=2, minibatches=2, hidden=512, obs=(4, 256, 256), rnn_layers=2),
    "serx101": dict(arch="serx101", E=4, T=128, epochs=2, minibatches=2, hidden=512, obs=(4, 256, 256), rnn_layers=2),
    # NEXT-3: the paper's best agent, SE-ResNeXt101 + 2-layer 1024-d LSTM
    "serx101_1024": dict(arch="serx101", E=4, T=128, epochs=2, minibatches=2, hidden=1024, obs=(4, 256, 256),
                         rnn_layers=2),
    "stress": dict(arch="depth", E=16, T=128, epochs=2, minibatches=2, hidden=512, obs=(1, 64, 64),
                   preempt_p=60),
}


def bf16_exact(x):
    """Round fp32 values to the nearest bf16 (ties to even), returned as fp32: depth frames are
    delivered to the GPU as bf16, so the generator emits bf16-exact values and every
    consumer (oracle, kernels) sees the same numbers."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    u = (u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) & np.uint32(0xFFFF0000)
    return u.view(np.float32)


def depth_frames(rng, E, T, C=1, H=64, W=64):
    """Smooth depth-like frames in [0, 1]: 3 seeded low-frequency cosine fields drifting over time
    plus 5 % noise (DESIGN.md input recipe)."""
    yy, xx = np.meshgrid(np.linspace(0, 1, H), np.linspace(0, 1, W), indexing="ij")
    out = np.empty((E, T, C, H, W), np.float32)
    for n in range(E):
        k = rng.uniform(0.5, 3.0, (3, 2))
        ph = rng.uniform(0, 2 * np.pi, 3)
        drift = rng.uniform(-0.05, 0.05, 3)
        for t in range(T):
            f = sum(np.cos(2 * np.pi * (k[i, 0] * xx + k[i, 1] * yy) + ph[i] + drift[i] * t) for i in range(3))
            f = 0.5 + f / 6.0 + 0.05 * rng.standard_normal((H, W))
            out[n, t] = bf16_exact(np.clip(f, 0.0, 1.0))[None].repeat(C, axis=0)
    return out


def rgbd_frames(rng, E, T, H=256, W=256):
    """RGB-D frames [E][T][4][H][W]: RGB in [0, 255] (integer-valued, like camera bytes) and depth in
    [0, 1], each channel a drifting sum of 3 seeded low-frequency cosine fields + 5 % noise."""
    yy, xx = np.meshgrid(np.linspace(0, 1, H), np.linspace(0, 1, W), indexing="ij")
    out = np.empty((E, T, 4, H, W), np.float32)
    for n in range(E):
        for ch in range(4):
            k = rng.uniform(0.5, 3.0, (3, 2))
            ph = rng.uniform(0, 2 * np.pi, 3)
            drift = rng.uniform(-0.05, 0.05, 3)
            base = [2 * np.pi * (k[i, 0] * xx + k[i, 1] * yy) + ph[i] for i in range(3)]
            cb, sb = [np.cos(b) for b in base], [np.sin(b) for b in base]
            for t in range(T):
                f = sum(cb[i] * np.cos(drift[i] * t) - sb[i] * np.sin(drift[i] * t) for i in range(3))
                f = np.clip(0.5 + f / 6.0 + 0.05 * rng.standard_normal((H, W)), 0.0, 1.0)
                out[n, t, ch] = np.rint(255.0 * f) if ch < 3 else bf16_exact(f)
    return out


def ld_for(T):
    return (T + 1 + 3) // 4 * 4


def _rng(seed, *keys):
    ss = np.random.SeedSequence([int(seed)] + [int(k) for k in keys])
    return np.random.Generator(np.random.Philox(ss))


def rollout(E, T, seed, rank=0, iteration=0, length=None, hidden=512, ld=None, obs_shape=None, rnn_layers=1):
    """One rank's rollout.  `length` (int or [E]) truncates (preemption); default T.
    obs_shape (C, H, W) adds frames `obs` [E][T][C][H][W] (C = 4: RGB-D) and an LSTM cell state `c0`;
    recurrent states are [E][rnn_layers * hidden] (layer-major)."""
    ld = ld or ld_for(T)
    rng = _rng(seed, 1, rank, iteration)
    f32 = np.float32
    rew = np.zeros((E, ld), f32)
    val = np.zeros((E, ld), f32)
    done = np.zeros((E, ld), np.uint8)
    action = np.zeros((E, ld), np.int32)
    prev_action = np.zeros((E, ld), np.int32)
    mask = np.zeros((E, ld), f32)
    logp_old = np.zeros((E, ld), f32)
    goal = np.zeros((E, T, 3), f32)

    # episode state (vectorised over envs); start mid-episode
    d0 = rng.uniform(1.0, 20.0, E)
    d = d0 * rng.uniform(0.3, 1.0, E)
    theta = rng.uniform(-np.pi, np.pi, E)
    path = d0 - d
    age = rng.integers(0, 100, E)
    prev = rng.integers(0, NUM_ACTIONS, E)
    m_prev = np.ones(E)
    for t in range(T + 1):
        val[:, t] = (2.5 * np.exp(-d / 10.0) - 0.05 * d + rng.normal(0.0, 0.1, E)).astype(f32)
        if t == T:
            break
        goal[:, t, 0] = d
        goal[:, t, 1] = np.cos(theta)
        goal[:, t, 2] = np.sin(theta)
        prev_action[:, t] = prev
        mask[:, t] = m_prev
        # behaviour policy: [stop, forward, left, right]
        towards_left = theta > 0
        p = np.zeros((E, 4))
        near = d <= 0.2
        p[:, 0] = np.where(near, 0.97, 0.02)
        rest = 1.0 - p[:, 0]
        p[:, 1] = rest * 0.6 / 0.98
        p[:, 2] = rest * np.where(towards_left, 0.28, 0.10) / 0.98
        p[:, 3] = rest * np.where(towards_left, 0.10, 0.28) / 0.98
        u = rng.random(E)
        a = (u[:, None] > np.cumsum(p, axis=1)).sum(axis=1).clip(0, 3)
        action[:, t] = a
        logp_old[:, t] = np.log(p[np.arange(E), a]).astype(f32)
        d_old = d.copy()
        collide = rng.random(E) < 0.1
        fwd = (a == 1) & ~collide
        gx = d * np.cos(theta) - 0.25 * fwd
        gy = d * np.sin(theta)
        d = np.where(fwd, np.hypot(gx, gy), d)
        theta = np.where(fwd, np.arctan2(gy, gx), theta)
        theta = theta + np.where(a == 2, -np.pi / 18, 0.0) + np.where(a == 3, np.pi / 18, 0.0)
        theta = (theta + np.pi) % (2 * np.pi) - np.pi
        path = path + 0.25 * fwd
        r = -(d - d_old) - 0.01
        age = age + 1
        ended = (a == 0) | (age >= 500)
        success = (a == 0) & (d_old <= 0.2)
        spl = np.where(success, d0 / np.maximum(d0, np.maximum(path, 1e-6)), 0.0)
        r = r + 2.5 * spl
        rew[:, t] = r.astype(f32)
        done[:, t] = ended.astype(np.uint8)
        # resets
        nd0 = rng.uniform(1.0, 20.0, E)
        nth = rng.uniform(-np.pi, np.pi, E)
        d0 = np.where(ended, nd0, d0)
        d = np.where(ended, nd0, d)
        theta = np.where(ended, nth, theta)
        path = np.where(ended, 0.0, path)
        age = np.where(ended, 0, age)
        prev = np.where(ended, START_TOKEN, a)
        m_prev = np.where(ended, 0.0, 1.0)

    if length is None:
        length = T
    length = np.broadcast_to(np.asarray(length, dtype=np.int32), (E,)).copy()
    for n in range(E):
        L = int(length[n])
        for arr in (rew, done, action, prev_action, mask, logp_old):
            arr[n, L:] = 0
        val[n, L + 1:] = 0
        goal[n, L:] = 0
    h0 = rng.normal(0.0, 0.1, (E, rnn_layers * hidden)).astype(f32)
    out = dict(rew=rew, val=val, done=done, length=length, goal=goal, prev_action=prev_action,
               mask=mask, action=action, logp_old=logp_old, h0=h0, E=E, T=T, ld=ld)
    if obs_shape is not None:
        if obs_shape[0] == 4:
            obs = rgbd_frames(_rng(seed, 6, rank, iteration), E, T, *obs_shape[1:])
        else:
            obs = depth_frames(_rng(seed, 6, rank, iteration), E, T, *obs_shape)
        for n in range(E):
            obs[n, int(length[n]):] = 0
        out["obs"] = obs
        out["c0"] = rng.normal(0.0, 0.1, (E, rnn_layers * hidden)).astype(f32)
    return out


def init_params(entries, P, seed):
    """entries: [(offset, numel, fan_in)] -> fp32 [P]; fan_in > 0: U(-1/sqrt(fan_in), 1/sqrt(fan_in))
    (torch default), fan_in == 0: ones (GroupNorm gamma), fan_in < 0: zeros (GroupNorm beta)."""
    rng = _rng(seed, 2)
    out = np.zeros(P, np.float32)
    for off, n, fan_in in entries:
        if fan_in > 0:
            k = 1.0 / np.sqrt(fan_in)
            out[off:off + n] = rng.uniform(-k, k, n).astype(np.float32)
        elif fan_in == 0:
            out[off:off + n] = 1.0
    return out


def perms(seed, iteration, epochs, E, rank=0):
    """Epoch permutations of env ids, int32 [epochs][E] (input of step a4)."""
    rng = _rng(seed, 3, rank, iteration)
    return np.stack([rng.permutation(E).astype(np.int32) for _ in range(epochs)])


def straggler_costs(seed, N, T, homogeneous=False, lo=1.0, hi=20.0):
    """Per-rank per-step costs in ticks (>= 1): s_w log-uniform[lo, hi] with +-10% jitter."""
    rng = _rng(seed, 4)
    s = np.full(N, 10.0) if homogeneous else np.exp(rng.uniform(np.log(lo), np.log(hi), N))
    jit = rng.uniform(-0.1, 0.1, (N, T))
    return np.maximum(1, np.rint(s[:, None] * (1.0 + jit))).astype(np.int64)


def random_loss_inputs(M, seed, A=NUM_ACTIONS, scale=1.0):
    """Generic per-sample loss inputs (test fixtures for step a6)."""
    rng = _rng(seed, 5)
    f32 = np.float32
    return dict(logits=(rng.normal(0, scale, (M, A))).astype(f32),
                values=rng.normal(0, 1, M).astype(f32),
                actions=rng.integers(0, A, M).astype(np.int32),
                logp_old=np.log(rng.uniform(0.05, 0.95, M)).astype(f32),
                values_old=rng.normal(0, 1, M).astype(f32),
                returns=rng.normal(0, 1, M).astype(f32),
                adv=rng.normal(0, 1, M).astype(f32))


class PointGoalEnv:
    """E synthetic PointGoal episodes stepped by the policy's own actions (the collection side of
    NEXT-1; the same dynamics as rollout(): P:L195-223, P:L207 actions, P:L221 reward, P:L588 goal
    [d, cos th, sin th]).  Frames: per env and channel three drifting low-frequency cosine fields +
    5 % noise (depth in [0, 1], bf16-exact; RGB integer bytes), as in depth_frames / rgbd_frames.
    Episodes start fresh (mask 0, prev action = start token) and end on stop or after 500 steps."""

    def __init__(self, E, seed, rank=0, obs=None, H=64):
        self.E, self.obs_kind, self.H = E, obs, H
        self.rng = _rng(seed, 7, rank)
        rng = self.rng
        self.d0 = rng.uniform(1.0, 20.0, E)
        self.d = self.d0.copy()
        self.theta = rng.uniform(-np.pi, np.pi, E)
        self.path = np.zeros(E)
        self.age = np.zeros(E, np.int64)
        self.prev = np.full(E, START_TOKEN, np.int64)
        self.m_prev = np.zeros(E)
        self.C = 0 if obs is None else (4 if obs == "rgbd" else 1)
        if self.C:
            yy, xx = np.meshgrid(np.linspace(0, 1, H), np.linspace(0, 1, H), indexing="ij")
            self._xy = (xx, yy)
            self.k = rng.uniform(0.5, 3.0, (E, self.C, 3, 2))
            self.ph = rng.uniform(0, 2 * np.pi, (E, self.C, 3))
            self.drift = rng.uniform(-0.05, 0.05, (E, self.C, 3))

    def observe(self):
        """(goal [E][3], prev_action [E], mask [E], frames [E][C][H][W] float32 or None) of the current
        state (the same arrays until the next step())."""
        if getattr(self, "_obs", None) is not None:
            return self._obs
        goal = np.stack([self.d, np.cos(self.theta), np.sin(self.theta)], 1).astype(np.float32)
        frames = None
        if self.C:
            xx, yy = self._xy
            frames = np.empty((self.E, self.C, self.H, self.H), np.float32)
            for n in range(self.E):
                for ch in range(self.C):
                    f = sum(np.cos(2 * np.pi * (self.k[n, ch, i, 0] * xx + self.k[n, ch, i, 1] * yy) + self.ph[n, ch, i]
                                   + self.drift[n, ch, i] * self.age[n]) for i in range(3))
                    f = np.clip(0.5 + f / 6.0 + 0.05 * self.rng.standard_normal((self.H, self.H)), 0.0, 1.0)
                    rgb = self.C == 4 and ch < 3
                    frames[n, ch] = np.rint(255.0 * f) if rgb else bf16_exact(f)
        self._obs = (goal, self.prev.astype(np.int32), self.m_prev.astype(np.float32), frames)
        return self._obs

    def step(self, a):
        """actions [E] in {stop, forward, left, right} -> (reward [E] float32, done [E] uint8)."""
        a = np.asarray(a, np.int64)
        rng, E = self.rng, self.E
        self._obs = None
        d_old = self.d.copy()
        collide = rng.random(E) < 0.1
        fwd = (a == 1) & ~collide
        gx = self.d * np.cos(self.theta) - 0.25 * fwd
        gy = self.d * np.sin(self.theta)
        self.d = np.where(fwd, np.hypot(gx, gy), self.d)
        th = np.where(fwd, np.arctan2(gy, gx), self.theta)
        th = th + np.where(a == 2, -np.pi / 18, 0.0) + np.where(a == 3, np.pi / 18, 0.0)
        self.theta = (th + np.pi) % (2 * np.pi) - np.pi
        self.path = self.path + 0.25 * fwd
        r = -(self.d - d_old) - 0.01
        self.age = self.age + 1
        ended = (a == 0) | (self.age >= 500)
        success = (a == 0) & (d_old <= 0.2)
        r = r + 2.5 * np.where(success, self.d0 / np.maximum(self.d0, np.maximum(self.path, 1e-6)), 0.0)
        nd0 = rng.uniform(1.0, 20.0, E)
        nth = rng.uniform(-np.pi, np.pi, E)
        self.d0 = np.where(ended, nd0, self.d0)
        self.d = np.where(ended, nd0, self.d)
        self.theta = np.where(ended, nth, self.theta)
        self.path = np.where(ended, 0.0, self.path)
        self.age = np.where(ended, 0, self.age)
        self.prev = np.where(ended, START_TOKEN, a)
        self.m_prev = np.where(ended, 0.0, 1.0)
        return r.astype(np.float32), ended.astype(np.uint8)
