"""Clipped-surrogate + value(-clip) + entropy loss and its gradient (step a6).

Test infrastructure only.

P:L129-138 (sec.2, Eq. 2): J = E_t[min(r_t(theta) A_t, clip(r_t, 1-eps, 1+eps) A_t)],
r_t = pi_theta(a_t|o_t) / pi_theta_old(a_t|o_t).  The value and
entropy terms are not in the paper; readings Z3/Z4: c_v = 0.5 on
0.5*MSE, c_e = 0.01, eps = 0.2; value clipping (PPO2
form, eps_v = eps) behind a flag as BASELINE.json asks.  Tie conventions
(Z5) follow torch: binary min/max split the gradient 1/2-1/2 on equality,
clamp passes the gradient on the closed interval.

Per valid sample i (n = number of valid samples, each weighted 1/n -- the
per-worker mean of P:L171 "We weigh all worker's contributions ... equally"):
    lse = logsumexp(z_i); lp = z_{i,a} - lse; p = softmax(z_i)
    rho = exp(lp - lp_old); u = rho*A; c = clip(rho, 1-eps, 1+eps)*A
    L_pi = -(1/n) sum min(u, c)
    v_c = v_old + clip(v - v_old, -eps_v, eps_v)
    L_v = (1/n) sum 0.5*max((v-R)^2, (v_c-R)^2)        (0.5*(v-R)^2 without clip)
    H_i = -sum_a p_a log p_a
    L = L_pi + c_v L_v - c_e (1/n) sum H_i
"""
import numpy as np

STAT_NAMES = ("policy_loss", "value_loss", "entropy", "clip_frac", "approx_kl", "total")


def _min_grad(x, y):
    """d min(x,y) / d(x, y) with torch's 1/2-1/2 split on ties."""
    gx = np.where(x < y, 1.0, np.where(x == y, 0.5, 0.0))
    return gx, 1.0 - gx


def _max_grad(x, y):
    gx = np.where(x > y, 1.0, np.where(x == y, 0.5, 0.0))
    return gx, 1.0 - gx


def loss_and_grad(logits, values, actions, logp_old, values_old, returns, adv,
                  valid, eps=0.2, vclip_eps=0.2, c_v=0.5, c_e=0.01,
                  use_value_clip=True, mean_invstd=None):
    """logits [M][A]; the rest [M]; valid [M] bool.  Returns (stats, dlogits, dvalues)."""
    z = np.asarray(logits, dtype=np.float64)
    v = np.asarray(values, dtype=np.float64)
    act = np.asarray(actions).astype(np.int64)
    lpo = np.asarray(logp_old, dtype=np.float64)
    vo = np.asarray(values_old, dtype=np.float64)
    R = np.asarray(returns, dtype=np.float64)
    A = np.asarray(adv, dtype=np.float64)
    w = np.asarray(valid).astype(np.float64)
    M, nA = z.shape
    if mean_invstd is not None:
        A = (A - mean_invstd[0]) * mean_invstd[1]
    n = w.sum()
    zmax = z.max(axis=1, keepdims=True)
    lse = (zmax + np.log(np.exp(z - zmax).sum(axis=1, keepdims=True)))[:, 0]
    logp = z - lse[:, None]
    p = np.exp(logp)
    lp = logp[np.arange(M), act]
    rho = np.exp(lp - lpo)
    u = rho * A
    rc = np.clip(rho, 1.0 - eps, 1.0 + eps)
    c = rc * A
    surr = np.minimum(u, c)
    H = -(p * logp).sum(axis=1)

    e1 = v - R
    if use_value_clip:
        vc = vo + np.clip(v - vo, -vclip_eps, vclip_eps)
        e2 = vc - R
        lv = 0.5 * np.maximum(e1 * e1, e2 * e2)
    else:
        lv = 0.5 * e1 * e1

    L_pi = -(w * surr).sum() / n
    L_v = (w * lv).sum() / n
    Hm = (w * H).sum() / n
    stats = {
        "policy_loss": L_pi,
        "value_loss": L_v,
        "entropy": Hm,
        "clip_frac": (w * (np.abs(rho - 1.0) > eps)).sum() / n,
        "approx_kl": (w * (lpo - lp)).sum() / n,
        "total": L_pi + c_v * L_v - c_e * Hm,
    }

    # d L / d lp  (chain rule through u = rho*A, c = clip(rho)*A, rho = exp(lp - lpo))
    gu, gc = _min_grad(u, c)
    inside = ((rho >= 1.0 - eps) & (rho <= 1.0 + eps)).astype(np.float64)
    dsurr_drho = gu * A + gc * A * inside
    dlp = -(w / n) * dsurr_drho * rho
    onehot = np.zeros_like(z)
    onehot[np.arange(M), act] = 1.0
    dlogits = dlp[:, None] * (onehot - p)
    # entropy: dH/dz_a = -p_a (log p_a + H)
    dlogits += (c_e * w / n)[:, None] * p * (logp + H[:, None])

    if use_value_clip:
        g1, g2 = _max_grad(e1 * e1, e2 * e2)
        vin = (np.abs(v - vo) <= vclip_eps).astype(np.float64)
        dlv = g1 * e1 + g2 * e2 * vin
    else:
        dlv = e1
    dvalues = c_v * (w / n) * dlv
    return stats, dlogits, dvalues
