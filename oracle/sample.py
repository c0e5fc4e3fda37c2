"""Action sampling of the collection side (NEXT-1, "collect experience with pi_theta").
Test infrastructure only.

The categorical draw both sides implement (include/ddppo.h ddppo_policy_act): per env e a uniform
u = (splitmix64(seed * 0x9E3779B97F4A7C15 + counter * 0xD1B54A32D192ED03 + e) >> 40) * 2^-24; with
m = max z, w_a = exp(z_a - m), S = sum w (fp32, in action order), the action is the first a whose
running sum exceeds u * S; logp = (z_a - m) - log S.  The decision is taken in fp32, the kernels'
precision (the oracle's exp may differ from the device's expf by an ulp: a draw within rounding of
a cumulative boundary is a near-tie where both actions are correct).
"""
import numpy as np

from .transfer import GAMMA, M64, splitmix64

GAMMA2 = 0xD1B54A32D192ED03


def uniforms(seed, counter, E):
    return np.array([np.float32(splitmix64((seed * GAMMA + counter * GAMMA2 + e) & M64) >> 40) *
                     np.float32(2.0 ** -24) for e in range(E)], dtype=np.float32)


def sample(logits, seed, counter, greedy=False):
    """logits [E][A] (fp32) -> (actions [E] int, logp [E] fp32, margin [E]): margin = the distance of
    u*S to the nearest cumulative boundary, relative to S (near-ties are < ~1e-6)."""
    z = np.asarray(logits, dtype=np.float32)
    E, A = z.shape
    u = uniforms(seed, counter, E)
    acts = np.zeros(E, np.int64)
    logp = np.zeros(E, np.float32)
    margin = np.full(E, np.inf)
    for e in range(E):
        m = z[e].max()
        w = np.exp(z[e] - m).astype(np.float32)
        S = np.float32(0.0)
        for a in range(A):
            S = np.float32(S + w[a])
        if greedy:
            a_sel = int(np.argmax(z[e]))
        else:
            target = np.float32(u[e] * S)
            c = np.float32(0.0)
            a_sel = A - 1
            for a in range(A):
                c = np.float32(c + w[a])
                margin[e] = min(margin[e], abs(float(c) - float(target)) / float(S))
                if c > target:
                    a_sel = a
                    break
        acts[e] = a_sel
        logp[e] = np.float32((z[e, a_sel] - m) - np.log(S))
    return acts, logp, margin
