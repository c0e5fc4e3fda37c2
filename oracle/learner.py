"""One synchronous, decentralized DD-PPO learner step over N ranks (steps a2-a8, a10).

Test infrastructure only.  P:L162-169 (sec.3, Eq. 4): every worker computes
grad J^PPO on its own rollout, the gradients are AllReduce-averaged and the
same ParamUpdate is applied on every worker; P:L219 fixes the PPO schedule
(epochs x minibatches); P:L171 weighs every worker equally (per-worker mean
loss, then the mean over workers).  The N ranks are emulated in one process.
"""
import numpy as np

from . import advnorm, gae, minibatch, models, optim, ppo

DEFAULT_CFG = dict(gamma=0.99, tau=0.95, normalize_adv=True, adv_eps=1e-5,
                   clip_eps=0.2, vclip_eps=0.2, c_v=0.5, c_e=0.01, use_value_clip=True,
                   epochs=2, minibatches=2, lr=2.5e-4, beta1=0.9, beta2=0.999,
                   adam_eps=1e-8, max_grad_norm=0.5)


def minibatch_grad(arch, params, ro, adv, ret, envs, mean_invstd, cfg, hidden=512, adopt=None):
    """Local gradient and loss stats of one rank on one minibatch of envs.  `adopt(batch, cache)`
    (tests only) may replace the forward's discrete ReLU / max-pool decisions in `cache` before the
    backward (reading R6: near-ties decided by the kernels)."""
    L = np.asarray(ro["length"])[envs]
    T_run = int(L.max())
    batch = {"goal": ro["goal"][envs, :T_run], "prev_action": ro["prev_action"][envs, :T_run],
             "mask": ro["mask"][envs, :T_run], "h0": ro["h0"][envs]}
    if "obs" in ro:
        batch["obs"] = ro["obs"][envs, :T_run]
        batch["c0"] = ro["c0"][envs]
    logits, values, cache = models.forward(arch, params, batch, hidden=hidden)
    if adopt is not None:
        adopt(batch, cache)
    B = len(envs)
    valid = (np.arange(T_run)[None, :] < L[:, None])
    flat = lambda a: np.asarray(a)[..., :T_run].reshape(B * T_run)  # noqa: E731
    stats, dlog, dval = ppo.loss_and_grad(
        logits.reshape(B * T_run, -1), values.reshape(-1),
        flat(ro["action"][envs]), flat(ro["logp_old"][envs]), flat(ro["val"][envs]),
        flat(ret[envs]), flat(adv[envs]), valid.reshape(-1),
        eps=cfg["clip_eps"], vclip_eps=cfg["vclip_eps"], c_v=cfg["c_v"], c_e=cfg["c_e"],
        use_value_clip=cfg["use_value_clip"], mean_invstd=mean_invstd)
    g = models.backward(arch, params, cache, dlog.reshape(B, T_run, -1), dval.reshape(B, T_run), hidden=hidden,
                        freeze_encoder=bool(cfg.get("freeze_encoder")))
    return g, stats, (logits, values, dlog, dval)


def learner_step(arch, params, m, v, step, rollouts, perms, cfg=None, hidden=512, trace=None):
    """rollouts: list (one per rank) of synth rollout dicts; perms[r][e] = env permutation.

    Returns (params, m, v, step, info).  `step` is the number of Adam steps
    already taken (the next update uses step+1).
    """
    cfg = dict(DEFAULT_CFG, **(cfg or {}))
    N = len(rollouts)
    advs, rets, stats3 = [], [], []
    for ro in rollouts:
        a, r = gae.gae(ro["rew"], ro["val"], ro["done"], ro["length"], cfg["gamma"], cfg["tau"])
        T = ro["goal"].shape[1]
        pad = lambda x: np.pad(x, ((0, 0), (0, T - x.shape[1])))  # noqa: E731
        advs.append(pad(a))
        rets.append(pad(r))
        stats3.append(gae.adv_stats(a, ro["length"]))
    gstats = advnorm.combine(stats3)
    mis = advnorm.mean_invstd(gstats, cfg["adv_eps"]) if cfg["normalize_adv"] else None
    params = np.asarray(params, dtype=np.float64)
    # NEXT-4: cfg["freeze"] (bool [P]) and / or cfg["freeze_encoder"] (the enc.* tensors)
    freeze = cfg.get("freeze")
    if cfg.get("freeze_encoder"):
        from .transfer import encoder_mask
        enc = encoder_mask(arch, params.size, hidden=hidden)
        freeze = enc if freeze is None else (np.asarray(freeze, bool) | enc)
    m = np.asarray(m, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    mb_stats, norms = [], []
    for e in range(cfg["epochs"]):
        for j in range(cfg["minibatches"]):
            grads, sts = [], []
            for r, ro in enumerate(rollouts):
                envs = minibatch.minibatch_envs(perms[r][e], cfg["minibatches"], j)
                g, st, extra = minibatch_grad(arch, params, ro, advs[r], rets[r], envs, mis, cfg, hidden)
                grads.append(g)
                sts.append(st)
                if trace is not None:
                    trace.append(dict(epoch=e, mb=j, rank=r, grad=g, stats=st, params=params.copy(),
                                      logits=extra[0], values=extra[1], dlogits=extra[2], dvalues=extra[3]))
            gbar = optim.allreduce_mean(grads)
            step += 1
            params, m, v, gn = optim.adam_step(params, gbar, m, v, step, lr=cfg["lr"], beta1=cfg["beta1"],
                                               beta2=cfg["beta2"], eps=cfg["adam_eps"],
                                               max_grad_norm=cfg["max_grad_norm"], freeze=freeze)
            norms.append(gn)
            mb_stats.append({k: float(np.mean([s[k] for s in sts])) for k in ppo.STAT_NAMES})
    steps = int(sum(int(np.sum(ro["length"])) for ro in rollouts))
    info = dict(adv=advs, ret=rets, adv_stats=gstats, mean_invstd=mis, mb_stats=mb_stats,
                grad_norms=norms, steps=steps)
    return params, m, v, step, info
