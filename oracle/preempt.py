"""Preemption-threshold protocol (step a9).  Test infrastructure only.

P:L171 (sec.3): "the rollout collection stage of these stragglers is
preempted (forced to end early) once some percentage, p%, ... of the other
workers are finished collecting their rollout ... We ... limit the minimum
number of steps before preemption to one-fourth the maximum".  P:L176/P:L637:
the finished-worker count lives in a shared store; processes preempt
themselves.  Readings: Z9 K = ceil(p*N/100) in integer
arithmetic (alternate ceil(p*(N-1)/100), clamped >= 1, behind a flag);
Z10 min = ceil(T/4); Z11 poll after every step, a finish at tick t is
visible at tick t (inclusive), and a rank finishing exactly at t* counts.

Virtual time: rank w's step i costs c[w][i] >= 1 ticks, so step s (1-based)
completes at tick C_w(s) = sum_{i<s} c[w][i]; F_w = C_w(T).
"""
import numpy as np


def threshold_count(p_percent, N, other_workers=False):
    """K = ceil(p% * N) (or of N-1 'other' workers, clamped to >= 1)."""
    base = N - 1 if other_workers else N
    k = (int(p_percent) * base + 99) // 100
    return max(k, 1)


def min_steps(T, min_steps_override=0):
    return int(min_steps_override) if min_steps_override else (T + 3) // 4


def should_stop(my_steps, T, finished_count, K, min_s):
    """Decision a rank takes right after completing step `my_steps`."""
    if my_steps >= T:
        return True
    return my_steps >= min_s and finished_count >= K


def closed_form_lengths(costs, T, p_percent, other_workers=False, min_steps_override=0):
    """L_w for every rank from the per-step costs (integers >= 1), closed form.

    t* = K-th smallest F_w;  L_w = T if F_w <= t*, else
    min(T, max(min, s*_w)) with s*_w = min{s : C_w(s) >= t*}.
    """
    costs = np.asarray(costs, dtype=np.int64)
    N = costs.shape[0]
    K = threshold_count(p_percent, N, other_workers)
    ms = min_steps(T, min_steps_override)
    C = np.concatenate([np.zeros((N, 1), dtype=np.int64), np.cumsum(costs[:, :T], axis=1)], axis=1)
    F = C[:, T]
    tstar = np.sort(F)[K - 1]
    L = np.empty(N, dtype=np.int64)
    for w in range(N):
        if F[w] <= tstar:
            L[w] = T
        else:
            s_star = int(np.argmax(C[w] >= tstar))  # first s with C_w(s) >= t*
            L[w] = min(T, max(ms, s_star))
    return L


def simulate_ticks(costs, T, p_percent, other_workers=False, min_steps_override=0):
    """Tick-by-tick simulation of the allreduce protocol (independent of the closed form).

    Every tick: each active rank advances its current step; ranks whose step
    ends on this tick record it (a rank reaching T steps is 'finished').
    Then all ranks exchange {finished, active} (the allreduce); every rank
    that completed a step on this tick and is still active applies
    should_stop.  Loop until no rank is active.  Returns (L, ticks, polls)
    where polls[k] = (tick, finished_count, active_count).
    """
    costs = np.asarray(costs, dtype=np.int64)
    N = costs.shape[0]
    K = threshold_count(p_percent, N, other_workers)
    ms = min_steps(T, min_steps_override)
    steps = [0] * N
    elapsed = [0] * N
    active = [True] * N
    finished = [False] * N
    polls = []
    tick = 0
    while any(active):
        tick += 1
        just_done = [False] * N
        for w in range(N):
            if not active[w]:
                continue
            elapsed[w] += 1
            if elapsed[w] == costs[w][steps[w]]:
                steps[w] += 1
                elapsed[w] = 0
                just_done[w] = True
                if steps[w] == T:
                    finished[w] = True
        fin_count = sum(finished)
        for w in range(N):
            if just_done[w] and active[w]:
                if should_stop(steps[w], T, fin_count, K, ms):
                    active[w] = False
        polls.append((tick, fin_count, sum(active)))
    return np.array(steps, dtype=np.int64), tick, polls


def step_accounting(lengths, envs_per_rank, T):
    """(collected, preempted) experience steps: sum_w E*L_w and sum_w E*(T-L_w)."""
    L = np.asarray(lengths, dtype=np.int64)
    return int((envs_per_rank * L).sum()), int((envs_per_rank * (T - L)).sum())
