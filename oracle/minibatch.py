"""PPO minibatch partition (step a4).  Test infrastructure only.

P:L219: "performs 2 epochs of PPO with 2 mini-batches per epoch".  Reading
Z13: minibatches partition *environments* (whole trajectories,
needed by the recurrent policy), reshuffled every epoch; the epoch
permutation pi_e is an input drawn by the host (synth.perms), consumed
identically by the oracle and the GPU.
"""
import numpy as np


def minibatch_envs(perm, num_minibatches, j):
    perm = np.asarray(perm, dtype=np.int64)
    E = perm.shape[0]
    if E % num_minibatches:
        raise ValueError("num_minibatches must divide the env count (S:L155)")
    B = E // num_minibatches
    return perm[j * B:(j + 1) * B]


def samples(envs, length):
    """List of (env, t) sample ids of one minibatch, env-major."""
    return [(int(n), t) for n in envs for t in range(int(length[n]))]
