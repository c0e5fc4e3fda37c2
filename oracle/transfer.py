"""Transfer-learning learner mechanics (NEXT-4).  Test infrastructure only.

P:L401-416 (sec.6): "The visual encoder is initialized from PointGoalNav and frozen"; "critic
layers are reinitialized"; the differentiable neural controller is frozen and a planner is trained
through it (its gradient wrt the goal input: models.backward(extra=...)).  S:L86-94 (reinit_critic):
only the value-head parameters are resampled, every other entry bit-identical.

The resampling uses a counter-based generator both sides implement (include/ddppo.h,
ddppo_reinit_critic): element i of the value head (row num_actions of head.weight, i < fan_in; the
bias is i = fan_in) takes u = splitmix64(seed * 0x9E3779B97F4A7C15 + i) >> 40 (24 bits) and the value
(u * 2^-23 - 1) * (1 / sqrt(fan_in)) in fp32, i.e. the default initialiser U(+-1/sqrt(fan_in)).
"""
import numpy as np

from . import models

M64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15


def splitmix64(x):
    """The SplitMix64 output function (Steele, Lea, Flood 2014) on one 64-bit integer."""
    z = x & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def encoder_mask(arch, P, hidden=512):
    """bool [P]: the visual encoder's entries (enc.* tensors)."""
    offs, P_ = models.offsets(arch, hidden=hidden)
    assert P_ == P
    mask = np.zeros(P, bool)
    for k, (o, s) in offs.items():
        if k.startswith("enc."):
            mask[o:o + int(np.prod(s))] = True
    return mask


def reinit_critic(arch, params, m, v, seed, hidden=512, num_actions=models.NUM_ACTIONS):
    """Returns (params', m', v') as float32 with the value head resampled and its m / v zeroed."""
    p = np.array(params, dtype=np.float32, copy=True)
    m = np.array(m, dtype=np.float32, copy=True)
    v = np.array(v, dtype=np.float32, copy=True)
    offs, _ = models.offsets(arch, hidden=hidden)
    (ow, sw), (ob, _) = offs["head.weight"], offs["head.bias"]
    fan_in = sw[1]
    bound = np.float32(1.0) / np.sqrt(np.float32(fan_in))
    idx = [ow + num_actions * fan_in + i for i in range(fan_in)] + [ob + num_actions]
    for i, at in enumerate(idx):
        u = splitmix64(seed * GAMMA + i) >> 40
        p[at] = (np.float32(u) * np.float32(2.0 ** -23) - np.float32(1.0)) * bound
        m[at] = 0.0
        v[at] = 0.0
    return p, m, v
