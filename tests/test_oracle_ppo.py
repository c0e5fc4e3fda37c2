"""Pins for oracle.ppo (step a6): Eq.2 worked values, identities, finite differences, torch autograd."""
import json
import os

import numpy as np
import torch

import synth
from oracle import ppo

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _call(x, valid, **kw):
    return ppo.loss_and_grad(x["logits"], x["values"], x["actions"], x["logp_old"], x["values_old"],
                             x["returns"], x["adv"], valid, **kw)


def test_ratio_one_policy_loss_is_minus_mean_adv():
    x = synth.random_loss_inputs(64, 1)
    z = x["logits"].astype(np.float64)
    lse = np.log(np.exp(z).sum(1))
    x["logp_old"] = z[np.arange(64), x["actions"]] - lse
    st, _, _ = _call(x, np.ones(64, bool))
    assert abs(st["policy_loss"] + np.mean(x["adv"].astype(np.float64))) < 1e-12
    assert st["clip_frac"] == 0.0 and abs(st["approx_kl"]) < 1e-12


def test_eq2_worked_value():
    g = GOLD["ppo_ratio2_adv1_eps02"]
    x = dict(logits=np.zeros((1, 4)), values=np.zeros(1), actions=np.zeros(1, np.int32),
             logp_old=np.array([np.log(0.25) - np.log(g["rho"])]), values_old=np.zeros(1),
             returns=np.zeros(1), adv=np.array([g["adv"]]))
    st, _, _ = _call(x, np.ones(1, bool), eps=g["eps"])
    assert abs(-st["policy_loss"] - g["surrogate"]) < 1e-12
    assert st["clip_frac"] == 1.0


def test_uniform_entropy():
    g = GOLD["entropy_uniform4"]
    x = synth.random_loss_inputs(8, 2)
    x["logits"] = np.zeros((8, 4))
    st, _, _ = _call(x, np.ones(8, bool))
    assert abs(st["entropy"] - g["entropy"]) < 1e-14


def test_clip_bound_property():
    """Eq.2's min makes every sample's contribution a pessimistic bound: <= u = rho*A for either
    sign of A, with equality inside [1-eps, 1+eps].  (S:L98 words the A<0 case as '>='; that is
    not a property of Eq.2 -- rho < 1-eps with A < 0 gives c < u.)"""
    x = synth.random_loss_inputs(256, 3, scale=2.0)
    for i in range(256):
        xi = {k: v[i:i + 1] for k, v in x.items()}
        st, _, _ = _call(xi, np.ones(1, bool))
        z = xi["logits"][0].astype(np.float64)
        lp = z[xi["actions"][0]] - np.log(np.exp(z).sum())
        u = np.exp(lp - xi["logp_old"][0]) * xi["adv"][0]
        contrib = -st["policy_loss"]
        rho = np.exp(lp - xi["logp_old"][0])
        assert contrib <= u + 1e-12
        if 0.8 <= rho <= 1.2:
            assert abs(contrib - u) < 1e-12


def _torch_loss(x, valid, eps, vclip, c_v, c_e, use_vc, mis):
    t = lambda a: torch.tensor(np.asarray(a, dtype=np.float64))  # noqa: E731
    z = t(x["logits"]).requires_grad_(True)
    v = t(x["values"]).requires_grad_(True)
    A = t(x["adv"])
    if mis is not None:
        A = (A - mis[0]) * mis[1]
    w = t(valid.astype(np.float64))
    n = w.sum()
    logp = torch.log_softmax(z, dim=1)
    lp = logp.gather(1, torch.tensor(x["actions"], dtype=torch.long)[:, None])[:, 0]
    rho = torch.exp(lp - t(x["logp_old"]))
    surr = torch.min(rho * A, torch.clamp(rho, 1 - eps, 1 + eps) * A)
    R = t(x["returns"])
    vo = t(x["values_old"])
    if use_vc:
        vc = vo + torch.clamp(v - vo, -vclip, vclip)
        lv = 0.5 * torch.max((v - R) ** 2, (vc - R) ** 2)
    else:
        lv = 0.5 * (v - R) ** 2
    H = -(logp.exp() * logp).sum(1)
    L = -(w * surr).sum() / n + c_v * (w * lv).sum() / n - c_e * (w * H).sum() / n
    L.backward()
    return float(L), z.grad.numpy(), v.grad.numpy()


def test_matches_torch_autograd_fp64_including_ties():
    for seed in range(40):
        x = synth.random_loss_inputs(48, 100 + seed, scale=1.5)
        x = {k: v.astype(np.float64) if v.dtype != np.int32 else v for k, v in x.items()}
        # force exact ties: rho == 1 and v == v_old on some samples
        z = x["logits"]
        lse = np.log(np.exp(z).sum(1))
        x["logp_old"][:8] = z[np.arange(8), x["actions"][:8]] - lse[:8]
        x["values_old"][8:14] = x["values"][8:14]
        valid = np.ones(48, bool)
        valid[40:] = False
        for use_vc in (True, False):
            mis = (0.1, 1.3) if seed % 2 else None
            st, dz, dv = _call(x, valid, use_value_clip=use_vc, mean_invstd=mis)
            L, tz, tv = _torch_loss(x, valid, 0.2, 0.2, 0.5, 0.01, use_vc, mis)
            assert abs(st["total"] - L) < 1e-12
            assert np.max(np.abs(dz - tz)) < 1e-13 and np.max(np.abs(dv - tv)) < 1e-13


def test_central_finite_differences():
    """h = 1e-5 central differences, samples away from the clip / max kinks."""
    x = synth.random_loss_inputs(12, 7)
    x = {k: v.astype(np.float64) if v.dtype != np.int32 else v for k, v in x.items()}
    valid = np.ones(12, bool)
    _, dz, dv = _call(x, valid)
    h = 1e-5
    for i in range(12):
        for a in range(4):
            xp = {k: v.copy() for k, v in x.items()}
            xm = {k: v.copy() for k, v in x.items()}
            xp["logits"][i, a] += h
            xm["logits"][i, a] -= h
            fd = (_call(xp, valid)[0]["total"] - _call(xm, valid)[0]["total"]) / (2 * h)
            assert abs(fd - dz[i, a]) < 1e-7
        xp = {k: v.copy() for k, v in x.items()}
        xm = {k: v.copy() for k, v in x.items()}
        xp["values"][i] += h
        xm["values"][i] -= h
        fd = (_call(xp, valid)[0]["total"] - _call(xm, valid)[0]["total"]) / (2 * h)
        assert abs(fd - dv[i]) < 1e-7
