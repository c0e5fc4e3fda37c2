"""Gradient AllReduce-mean + global-norm clip + Adam (step a8).  Test infrastructure only.

P:L150-158 (sec.3, Eq. 3): theta^{k+1}_n = ParamUpdate(theta^k_n,
(1/N) sum_i grad^k_i); P:L162-169 (Eq. 4) applies it to grad J^PPO.
P:L219: "We use Adam with a learning rate of 2.5e-4".  Readings:
Z14 beta1 0.9, beta2 0.999, eps 1e-8, bias-corrected PyTorch form,
constant lr; Z15 global L2 clip 0.5 on the *averaged* gradient (S:L80,
S:L107), coef = min(1, max_norm / (||g|| + 1e-6)); the mean is
a rank-ordered sum then one multiply by 1/N.
"""
import numpy as np


def allreduce_mean(grads):
    """(1/N) * sum_{n=0..N-1} g_n, summed in ascending rank order."""
    acc = np.zeros_like(np.asarray(grads[0], dtype=np.float64))
    for g in grads:
        acc = acc + np.asarray(g, dtype=np.float64)
    return acc * (1.0 / len(grads))


def clip_coef(g, max_norm):
    total = np.sqrt(np.sum(np.asarray(g, dtype=np.float64) ** 2))
    return min(1.0, max_norm / (total + 1e-6)), total


def adam_step(params, grad, m, v, step, lr=2.5e-4, beta1=0.9, beta2=0.999,
              eps=1e-8, max_grad_norm=0.5, freeze=None):
    """One step; `step` is the 1-based step index of this update.

    Returns (params', m', v', grad_norm_before_clip).  Frozen entries
    (freeze[i] true) keep params, m, v bit-identical.
    """
    p = np.asarray(params, dtype=np.float64).copy()
    g = np.asarray(grad, dtype=np.float64)
    m = np.asarray(m, dtype=np.float64).copy()
    v = np.asarray(v, dtype=np.float64).copy()
    if max_grad_norm is not None and max_grad_norm > 0:
        coef, total = clip_coef(g, max_grad_norm)
    else:
        coef, total = 1.0, np.sqrt(np.sum(g * g))
    g = g * coef
    upd = np.ones(p.shape, dtype=bool) if freeze is None else ~np.asarray(freeze, dtype=bool)
    m_new = beta1 * m + (1.0 - beta1) * g
    v_new = beta2 * v + (1.0 - beta2) * g * g
    bc1 = 1.0 - beta1 ** step
    bc2 = 1.0 - beta2 ** step
    denom = np.sqrt(v_new) / np.sqrt(bc2) + eps
    p_new = p - (lr / bc1) * m_new / denom
    p = np.where(upd, p_new, p)
    m = np.where(upd, m_new, m)
    v = np.where(upd, v_new, v)
    return p, m, v, total
