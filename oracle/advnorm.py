"""Advantage normalisation (step a3).  Test infrastructure only.

The paper does NOT normalise advantages ("Unlike popular
implementations of PPO, we do not normalize advantages"); BASELINE.json's
north_star puts it on the hot path as "a block reduction plus a cross-rank
allreduce of sum and sum-of-squares".  Readings Z1/Z2: a flag;
statistics are global over ranks and count-weighted (preemption makes the
per-rank counts differ), unbiased (n-1), eps = 1e-5 added to sigma.
"""
import numpy as np


def combine(stats_per_rank):
    """Allreduce(sum) of the per-rank {S, Q, n} triples, rank order 0..N-1."""
    tot = np.zeros(3)
    for s in stats_per_rank:
        tot = tot + np.asarray(s, dtype=np.float64)
    return tot


def mean_invstd(global_stats, eps=1e-5):
    """mu = S/n; sigma^2 = (Q - n mu^2)/(n-1); returns (mu, 1/(sigma+eps))."""
    S, Q, n = (float(x) for x in global_stats)
    mu = S / n
    var = (Q - n * mu * mu) / (n - 1.0) if n > 1 else 0.0
    var = max(var, 0.0)
    return mu, 1.0 / (np.sqrt(var) + eps)


def normalize(adv, mu, invstd):
    return (np.asarray(adv, dtype=np.float64) - mu) * invstd
