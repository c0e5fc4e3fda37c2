"""B200-native DD-PPO learner step (arXiv 1911.00357) behind the C ABI of include/ddppo.h.

The functions below carry the C names and only marshal arguments; torch is used for
device memory, streams and process groups.  See DESIGN.md.
"""
import ctypes

import numpy as np

from . import _lib
from ._lib import (ActBatch, ARCH_DEPTH, ARCH_GPS, ARCH_RGBD, ARCH_TOY, AdamCfg, Batch, DdppoError, LearnerCfg, LossCfg, LossInputs, ModelDesc,
                   PreemptCfg, Rollout, TensorInfo, check, dptr, f32, f64, i32, lib, u8)

__all__ = ["Context", "model_desc", "param_layout", "ddppo_gae", "ddppo_adv_norm", "ddppo_policy_fwd",
           "ddppo_policy_bwd", "ddppo_ppo_loss_grad", "ddppo_grad_allreduce_step", "ddppo_preempt_poll",
           "ddppo_preempt_decide", "ddppo_preempt_threshold", "ddppo_allreduce_counts", "ddppo_learner_step",
           "DdppoError", "lib"]


def _stream(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def model_desc(arch, hidden=None, num_actions=4):
    arch_id = {"toy": ARCH_TOY, "gps": ARCH_GPS, "depth": ARCH_DEPTH, "rgbd": ARCH_RGBD,
               "serx50": _lib.ARCH_SERX50, "serx101": _lib.ARCH_SERX101}.get(arch, arch)
    if hidden is None:
        hidden = 64 if arch_id == ARCH_TOY else 512
    d = ModelDesc()
    d.arch, d.hidden, d.num_actions = arch_id, hidden, num_actions
    return d


def param_count(desc):
    P = ctypes.c_int64()
    check("ddppo_model_param_count", lib.ddppo_model_param_count(ctypes.byref(desc), ctypes.byref(P)))
    return P.value


def param_layout(desc):
    """[(name, offset, shape, fan_in)] in the documented order."""
    n = ctypes.c_int()
    check("ddppo_model_param_layout", lib.ddppo_model_param_layout(ctypes.byref(desc), None, 0, ctypes.byref(n)))
    arr = (TensorInfo * n.value)()
    check("ddppo_model_param_layout", lib.ddppo_model_param_layout(ctypes.byref(desc), arr, n.value, ctypes.byref(n)))
    return [(t.name.decode(), t.offset, tuple(t.shape[:t.ndim]), t.fan_in) for t in arr]


def workspace_size(desc, max_B, T):
    b = ctypes.c_size_t()
    check("ddppo_workspace_size", lib.ddppo_workspace_size(ctypes.byref(desc), max_B, T, ctypes.byref(b)))
    return b.value


def learner_workspace_size(desc, E, T, ld, minibatches, epochs):
    b = ctypes.c_size_t()
    check("ddppo_learner_workspace_size",
          lib.ddppo_learner_workspace_size(ctypes.byref(desc), E, T, ld, minibatches, epochs, ctypes.byref(b)))
    return b.value


def get_unique_id():
    buf = (ctypes.c_uint8 * 128)()
    check("ddppo_get_unique_id", lib.ddppo_get_unique_id(buf))
    return bytes(buf)


class Context:
    """Owns a ddppo_ctx (NCCL communicator + scratch) for one rank."""

    def __init__(self, rank=0, world=1, unique_id=None, device=0):
        self.rank, self.world, self.device = rank, world, device
        h = ctypes.c_void_p()
        idbuf = None
        if world > 1:
            idbuf = (ctypes.c_uint8 * 128).from_buffer_copy(unique_id)
        code = lib.ddppo_ctx_create(rank, world, idbuf, device, ctypes.byref(h))
        check("ddppo_ctx_create", code)
        self.h = h

    def close(self):
        if self.h:
            lib.ddppo_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, stream=None):
        check("ddppo_check", lib.ddppo_check(self.h, _stream(stream)), self.h)


def _call(ctx, fn, *args):
    check(fn, getattr(lib, fn)(ctx.h, *args), ctx.h)


def ddppo_gae(ctx, rew, val, done, length, E, T, ld, gamma, tau, adv, ret, stats3=None, stream=None):
    _call(ctx, "ddppo_gae", f32(rew), f32(val), u8(done), i32(length), E, T, ld, gamma, tau, f32(adv),
          f32(ret), f64(stats3), _stream(stream))


def ddppo_adv_norm(ctx, stats3, eps, mean_invstd, stream=None):
    _call(ctx, "ddppo_adv_norm", f64(stats3), eps, f32(mean_invstd), _stream(stream))


BATCH_FREEZE_ENCODER = 1


def make_batch(goal, prev_action, mask, h0, length, env_idx, E, T, ld, B, T_run, n_valid, obs=None, c0=None,
               obs_rgb=None, dgoal=None, freeze_encoder=False):
    """obs: depth frames (torch.bfloat16); obs_rgb: RGB camera bytes (torch.uint8, RGB-D only);
    dgoal: optional [B*T_run][3] output of the visual agents' backward (dL/d goal input);
    freeze_encoder: the visual encoder is frozen (no encoder backward, its gradient 0)."""
    b = Batch()
    b.goal, b.prev_action, b.mask, b.h0 = f32(goal), i32(prev_action), f32(mask), f32(h0)
    b.len, b.env_idx = i32(length), i32(env_idx)
    b.E, b.T, b.ld, b.B, b.T_run, b.n_valid = E, T, ld, B, T_run, n_valid
    b.obs = dptr(obs, "bfloat16") if obs is not None else None
    b.c0 = f32(c0) if c0 is not None else None
    b.obs_rgb = u8(obs_rgb) if obs_rgb is not None else None
    b.dgoal = f32(dgoal) if dgoal is not None else None
    b.flags = BATCH_FREEZE_ENCODER if freeze_encoder else 0
    b._keep = (goal, prev_action, mask, h0, length, env_idx, obs, c0, obs_rgb, dgoal)  # raw pointers held
    return b


def visual_obs(obs, rgbd):
    """A synth-style float frame array [E][T][C][H][W] -> the ABI's observation tensors (host, torch):
    {"obs": depth channel as bf16, "obs_rgb": RGB channels as uint8 (RGB-D only)} -- dtype
    marshalling only (the generator's depth values are bf16-exact and its RGB values integers)."""
    import torch
    a = np.asarray(obs, dtype=np.float32)
    out = {"obs": torch.from_numpy(np.ascontiguousarray(a[:, :, 3:4] if rgbd else a)).to(torch.bfloat16)}
    if rgbd:
        out["obs_rgb"] = torch.from_numpy(np.ascontiguousarray(a[:, :, :3]).astype(np.uint8))
    return out


def ddppo_policy_fwd(ctx, desc, params, batch, logits, values, ws, stream=None):
    _call(ctx, "ddppo_policy_fwd", ctypes.byref(desc), f32(params), ctypes.byref(batch), f32(logits),
          f32(values), dptr(ws), ws.numel() * ws.element_size(), _stream(stream))


def ddppo_policy_bwd(ctx, desc, params, batch, dlogits, dvalues, grad, ws, stream=None):
    _call(ctx, "ddppo_policy_bwd", ctypes.byref(desc), f32(params), ctypes.byref(batch), f32(dlogits),
          f32(dvalues), f32(grad), dptr(ws), ws.numel() * ws.element_size(), _stream(stream))


def loss_cfg(clip_eps=0.2, vclip_eps=0.2, c_v=0.5, c_e=0.01, use_value_clip=True, normalize_adv=True):
    c = LossCfg()
    c.clip_eps, c.vclip_eps, c.c_v, c.c_e = clip_eps, vclip_eps, c_v, c_e
    c.use_value_clip, c.normalize_adv = int(use_value_clip), int(normalize_adv)
    return c


def ddppo_ppo_loss_grad(ctx, logits, values, batch, action, logp_old, value_old, ret, adv, mean_invstd, cfg,
                        dlogits, dvalues, stats, stream=None):
    li = LossInputs()
    li.action, li.logp_old, li.value_old, li.ret, li.adv = (i32(action), f32(logp_old), f32(value_old),
                                                            f32(ret), f32(adv))
    _call(ctx, "ddppo_ppo_loss_grad", f32(logits), f32(values), ctypes.byref(batch), ctypes.byref(li),
          f32(mean_invstd), ctypes.byref(cfg), f32(dlogits), f32(dvalues), f32(stats), _stream(stream))


def adam_cfg(step, lr=2.5e-4, beta1=0.9, beta2=0.999, eps=1e-8, max_grad_norm=0.5):
    c = AdamCfg()
    c.lr, c.beta1, c.beta2, c.eps, c.max_grad_norm, c.step = lr, beta1, beta2, eps, max_grad_norm, step
    return c


def ddppo_grad_allreduce_step(ctx, grad, params, m, v, cfg, freeze_mask=None, grad_norm=None, stream=None):
    _call(ctx, "ddppo_grad_allreduce_step", f32(grad), f32(params), f32(m), f32(v), u8(freeze_mask),
          params.numel(), ctypes.byref(cfg), f32(grad_norm), _stream(stream))


def preempt_cfg(p_percent, T, min_steps=0, other_workers=False):
    c = PreemptCfg()
    c.p_percent, c.T, c.min_steps, c.other_workers = p_percent, T, min_steps, int(other_workers)
    return c


def ddppo_preempt_threshold(cfg, world):
    K, ms = ctypes.c_int(), ctypes.c_int()
    check("ddppo_preempt_threshold", lib.ddppo_preempt_threshold(ctypes.byref(cfg), world, ctypes.byref(K),
                                                                 ctypes.byref(ms)))
    return K.value, ms.value


def ddppo_preempt_decide(cfg, world, my_steps, finished_count):
    out = ctypes.c_int()
    check("ddppo_preempt_decide", lib.ddppo_preempt_decide(ctypes.byref(cfg), world, my_steps, finished_count,
                                                           ctypes.byref(out)))
    return bool(out.value)


def ddppo_preempt_poll(ctx, my_steps, finished, active, cfg):
    stop, fin, act = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    _call(ctx, "ddppo_preempt_poll", my_steps, int(finished), int(active), ctypes.byref(cfg), ctypes.byref(stop),
          ctypes.byref(fin), ctypes.byref(act))
    return bool(stop.value), fin.value, act.value


def ddppo_allreduce_counts(ctx, values):
    arr = np.ascontiguousarray(np.asarray(values, dtype=np.int64))
    _call(ctx, "ddppo_allreduce_counts", arr.ctypes.data, arr.size)
    return arr


def learner_cfg(epochs=2, minibatches=2, gamma=0.99, tau=0.95, normalize_adv=True, adv_eps=1e-5, loss=None,
                adam=None):
    c = LearnerCfg()
    c.gamma, c.tau, c.adv_eps, c.normalize_adv = gamma, tau, adv_eps, int(normalize_adv)
    c.epochs, c.minibatches = epochs, minibatches
    c.loss = loss or loss_cfg(normalize_adv=normalize_adv)
    c.adam = adam or adam_cfg(0)
    return c


def ddppo_debug_gemm_bf16(ctx, A, sam, sak, B, sbn, sbk, C, ldc, M, N, K, splits=1, partial=None, prec=1,
                          stream=None):
    """C[m][n] = sum_k A(m,k) B(n,k) on the tcgen05 path (A, B, C fp32 CUDA tensors; strides in elements)."""
    _call(ctx, "ddppo_debug_gemm_bf16", f32(A), sam, sak, f32(B), sbn, sbk, f32(C), ldc, M, N, K, splits,
          f32(partial), prec, _stream(stream))


def ddppo_debug_conv2d(ctx, x, w, F, H, W, Ci, Co, k, s, p, y=None, dy=None, dx=None, dw=None, stream=None):
    """Depth encoder convolution (NHWC activations, [Co][Ci][k][k] weights) on the tcgen05 path."""
    import torch
    need = ctypes.c_size_t()
    args = (f32(x), f32(w), F, H, W, Ci, Co, k, s, p, f32(y), f32(dy), f32(dx), f32(dw))
    _call(ctx, "ddppo_debug_conv2d", *args, None, 0, ctypes.byref(need), _stream(stream))
    scratch = torch.empty(need.value // 4 + 64, dtype=torch.float32, device=x.device)
    _call(ctx, "ddppo_debug_conv2d", *args, f32(scratch), scratch.numel() * 4, None, _stream(stream))
    return scratch  # keep alive until the stream has run


def ddppo_debug_groupnorm(ctx, y, gamma, beta, F, HW, C, relu, z, stats, residual=None, dz=None, dy=None,
                          dgamma=None, dbeta=None, stream=None):
    import torch
    scratch = torch.empty(4 * F * HW * C + 64 * F + 1024, dtype=torch.float32, device=y.device)
    _call(ctx, "ddppo_debug_groupnorm", f32(y), f32(gamma), f32(beta), f32(residual), F, HW, C, int(relu), f32(z),
          f32(stats), f32(dz), f32(dy), f32(dgamma), f32(dbeta), f32(scratch), _stream(stream))
    return scratch


def ddppo_debug_depth_decisions(ctx, desc, batch, ws, stream=None):
    """uint8 CUDA tensor of the Depth forward's ReLU masks / max-pool argmax (include/ddppo.h order)."""
    import torch
    n = ctypes.c_int64()
    _call(ctx, "ddppo_debug_depth_decisions", ctypes.byref(desc), ctypes.byref(batch), dptr(ws), None, 0,
          ctypes.byref(n), _stream(stream))
    out = torch.zeros(n.value, dtype=torch.uint8, device=ws.device)
    _call(ctx, "ddppo_debug_depth_decisions", ctypes.byref(desc), ctypes.byref(batch), dptr(ws), u8(out), n.value,
          None, _stream(stream))
    return out


def ddppo_debug_maxpool(ctx, x, F, H, W, C, y, arg, dy=None, dx=None, stream=None):
    _call(ctx, "ddppo_debug_maxpool", f32(x), F, H, W, C, f32(y), u8(arg), f32(dy), f32(dx), _stream(stream))


def profile_enable(ctx, on=True):
    _call(ctx, "ddppo_profile_enable", int(on))


def profile_read(ctx, reset=False):
    """{family: (ms, launches, flops)} accumulated since the last reset (blocking)."""
    n = len(_lib.KERNEL_FAMILIES)
    ms = (ctypes.c_double * n)()
    la = (ctypes.c_int64 * n)()
    fl = (ctypes.c_double * n)()
    _call(ctx, "ddppo_profile_read", ms, la, int(reset))
    _call(ctx, "ddppo_profile_flops", fl, int(reset))
    return {k: (ms[i], la[i], fl[i]) for i, k in enumerate(_lib.KERNEL_FAMILIES)}


def ddppo_rollout_steps(host_len, T):
    """a10 input: sum_e min(len_e, T) of an int32 host array (computed in the C library)."""
    ln = np.ascontiguousarray(np.asarray(host_len, dtype=np.int32))
    out = ctypes.c_int64()
    r = _lib.lib.ddppo_rollout_steps(ln.ctypes.data, int(ln.size), int(T), ctypes.byref(out))
    if r != 0:
        raise DdppoError("ddppo_rollout_steps", r, "lengths must be >= 0, E >= 1, T >= 1")
    return int(out.value)


def profile_smem_bytes(ctx, reset=False):
    """{family: shared-memory bytes moved by the tensor-core conv kernels} since the last reset."""
    n = len(_lib.KERNEL_FAMILIES)
    b = (ctypes.c_double * n)()
    _call(ctx, "ddppo_profile_smem_bytes", b, int(reset))
    return {k: b[i] for i, k in enumerate(_lib.KERNEL_FAMILIES)}


def ddppo_set_graphs(ctx, enable=True):
    """CUDA-graph replay of ddppo_learner_step (default on; eager while profiling)."""
    _call(ctx, "ddppo_set_graphs", int(enable))


def ddppo_learner_register(ctx, ws):
    """Collective: expose this learner workspace to all ranks (a8 over NVLink peer memory)."""
    _call(ctx, "ddppo_learner_register", dptr(ws), ws.numel() * ws.element_size())


def ddppo_learner_step(ctx, desc, ro, cfg, params, m, v, adv, ret, stats_out, ws, stream=None):
    """ro: Rollout struct (device pointers + host lengths/perms). Returns the new Adam step count."""
    step = ctypes.c_int32()
    _call(ctx, "ddppo_learner_step", ctypes.byref(desc), ctypes.byref(ro), ctypes.byref(cfg), f32(params), f32(m),
          f32(v), f32(adv), f32(ret), f32(stats_out), dptr(ws), ws.numel() * ws.element_size(),
          ctypes.byref(step), _stream(stream))
    return step.value


def ddppo_set_a8_mode(ctx, mode):
    """"sharded" (reduce-scatter -> shard Adam -> all-gather), "allread" (v1) or "auto" (default)."""
    _call(ctx, "ddppo_set_a8_mode", {"sharded": _lib.A8_SHARDED, "allread": _lib.A8_ALLREAD,
                                     "auto": _lib.A8_AUTO}.get(mode, mode))


def _ptr_array(ts):
    arr = (ctypes.c_void_p * len(ts))()
    for i, t in enumerate(ts):
        arr[i] = f32(t)
    return arr


def ddppo_debug_peer_a8(ctx, mode, grads, params, m, v, cfg, gsum, stream=None):
    """Single-device emulation of the peer-memory a8 over N = len(grads) ranks (lists of [P] tensors)."""
    import torch
    mode = {"sharded": _lib.A8_SHARDED, "allread": _lib.A8_ALLREAD}.get(mode, mode)
    N, P = len(grads), params[0].numel()
    arrs = [_ptr_array(x) for x in (grads, params, m, v, gsum)]
    need = ctypes.c_size_t()
    _call(ctx, "ddppo_debug_peer_a8", N, mode, *arrs[:4], P, ctypes.byref(cfg), arrs[4], None, 0,
          ctypes.byref(need), _stream(stream))
    scratch = torch.empty(need.value, dtype=torch.uint8, device=params[0].device)
    _call(ctx, "ddppo_debug_peer_a8", N, mode, *arrs[:4], P, ctypes.byref(cfg), arrs[4], dptr(scratch),
          need.value, None, _stream(stream))
    return scratch


def ddppo_debug_peer_counts(ctx, vals):
    """vals [N][n] int64 -> [N][n]: each emulated rank's rank-ordered sums (blocking)."""
    import torch
    v = np.ascontiguousarray(np.asarray(vals, dtype=np.int64))
    N, n = v.shape
    out = np.zeros_like(v)
    need = ctypes.c_size_t()
    _call(ctx, "ddppo_debug_peer_counts", N, v.ctypes.data, n, out.ctypes.data, None, 0, ctypes.byref(need))
    scratch = torch.empty(need.value, dtype=torch.uint8, device=f"cuda:{ctx.device}")
    _call(ctx, "ddppo_debug_peer_counts", N, v.ctypes.data, n, out.ctypes.data, dptr(scratch), need.value, None)
    return out


def ddppo_layout_hash(desc, E, T, ld, minibatches, epochs):
    h = ctypes.c_uint64()
    check("ddppo_layout_hash", lib.ddppo_layout_hash(ctypes.byref(desc), E, T, ld, minibatches, epochs,
                                                     ctypes.byref(h)))
    return h.value


def ddppo_layout_check(ctx, desc, E, T, ld, minibatches, epochs):
    """Collective: DdppoError(protocol) unless every rank has the same layout hash."""
    _call(ctx, "ddppo_layout_check", ctypes.byref(desc), E, T, ld, minibatches, epochs)


def ddppo_set_conv_engine(ctx, engine):
    """"tma" (TMA-fed warp-specialised tcgen05 convolutions, default) or "cpasync" (round-1 kernel)."""
    _call(ctx, "ddppo_set_conv_engine", {"cpasync": 0, "tma": 1}.get(engine, engine))


def ddppo_reinit_critic(ctx, desc, params, m, v, seed, stream=None):
    """Resample the value head with the documented counter-based generator."""
    _call(ctx, "ddppo_reinit_critic", ctypes.byref(desc), f32(params), f32(m), f32(v), int(seed), _stream(stream))


def act_workspace_size(desc, E):
    b = ctypes.c_size_t()
    check("ddppo_act_workspace_size", lib.ddppo_act_workspace_size(ctypes.byref(desc), E, ctypes.byref(b)))
    return b.value


def make_act_batch(goal, prev_action, mask, h_in, h_out, E, T, ld, t, seed, counter, obs=None, obs_rgb=None,
                   c_in=None, c_out=None, greedy=False):
    """Step t of E envs (rollout layout, see include/ddppo.h ddppo_act_batch)."""
    a = ActBatch()
    a.goal, a.prev_action, a.mask = f32(goal), i32(prev_action), f32(mask)
    a.obs = dptr(obs, "bfloat16") if obs is not None else None
    a.obs_rgb = u8(obs_rgb) if obs_rgb is not None else None
    a.E, a.T, a.ld, a.t = E, T, ld, t
    a.h_in, a.h_out = f32(h_in), f32(h_out)
    a.c_in = f32(c_in) if c_in is not None else None
    a.c_out = f32(c_out) if c_out is not None else None
    a.seed, a.counter, a.greedy = int(seed), int(counter), int(greedy)
    a._keep = (goal, prev_action, mask, obs, obs_rgb, h_in, h_out, c_in, c_out)
    return a


def ddppo_policy_act(ctx, desc, params, act_batch, actions, logp, values, ws, logits=None, stream=None):
    _call(ctx, "ddppo_policy_act", ctypes.byref(desc), f32(params), ctypes.byref(act_batch), i32(actions), f32(logp),
          f32(values), f32(logits), dptr(ws), ws.numel() * ws.element_size(), _stream(stream))


def ddppo_set_fwd_planes(ctx, planes):
    """Encoder forward operands: 2 = bf16 hi/lo planes (default), 1 = plain bf16."""
    _call(ctx, "ddppo_set_fwd_planes", int(planes))
