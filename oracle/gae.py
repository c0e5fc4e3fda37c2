"""GAE reverse-time scan (step a2).  Test infrastructure only (see oracle/__init__).

P:L218 (sec.4 Training): "We use PPO with Generalized Advantage Estimation
... discount factor gamma 0.99 ... GAE parameter tau 0.95".  The estimator
itself is the cited one:

    delta_t = r_t + gamma * V_{t+1} * (1 - done_t) - V_t
    A_t     = delta_t + gamma * tau * (1 - done_t) * A_{t+1},   A_L = 0
    R_t     = A_t + V_t                     (A_t = R_t - V_t)

Readings (Z6/Z8): done_t = "transition t ended the episode" and
masks both the bootstrap and the trace; rollouts cross episode boundaries;
a rollout truncated at length L (preemption) bootstraps from V_L, stored in
slot L of the value row.  Outputs for t >= L are 0.
"""
import numpy as np


def gae(rew, val, done, length, gamma, tau):
    """rew, done: [E][>=T]; val: [E][>=T+1]; length: [E] ints (<= T).

    Returns (adv, ret) as float64 [E][T] where T = max(length) (zeros past
    each env's length).  Loop over t backwards, vectorised over envs only.
    """
    rew = np.asarray(rew, dtype=np.float64)
    val = np.asarray(val, dtype=np.float64)
    done = np.asarray(done).astype(np.float64)
    length = np.asarray(length, dtype=np.int64)
    E = rew.shape[0]
    T = int(length.max()) if E else 0
    adv = np.zeros((E, T))
    ret = np.zeros((E, T))
    a_next = np.zeros(E)
    for t in range(T - 1, -1, -1):
        valid = t < length
        nd = 1.0 - done[:, t]
        delta = rew[:, t] + gamma * val[:, t + 1] * nd - val[:, t]
        a = delta + gamma * tau * nd * a_next
        a = np.where(valid, a, 0.0)
        adv[:, t] = a
        ret[:, t] = np.where(valid, a + val[:, t], 0.0)
        a_next = a
    return adv, ret


def adv_stats(adv, length):
    """Local {sum A, sum A^2, n} over the valid entries, float64 (step a3)."""
    adv = np.asarray(adv, dtype=np.float64)
    length = np.asarray(length, dtype=np.int64)
    T = adv.shape[1] if adv.ndim == 2 else 0
    valid = np.arange(T)[None, :] < length[:, None]
    a = adv[valid]
    return np.array([a.sum(), (a * a).sum(), float(valid.sum())])
