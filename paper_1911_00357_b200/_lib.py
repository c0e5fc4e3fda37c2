"""ctypes binding of libddppo.so (include/ddppo.h).  Argument marshalling only.

Every computation runs in the CUDA kernels behind the C ABI; there is no CPU fallback.
If libddppo.so is missing this module raises at import time.
"""
import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libddppo.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(there is no CPU fallback for the DD-PPO kernels)")

lib = ctypes.CDLL(LIB_PATH)

c_int, c_float, c_double, c_vp, c_i64 = ctypes.c_int, ctypes.c_float, ctypes.c_double, ctypes.c_void_p, ctypes.c_int64
c_i32, c_size = ctypes.c_int32, ctypes.c_size_t

STATUS = {0: "ok", 1: "config", 2: "numerical", 3: "protocol", 4: "comm", 5: "cuda", 6: "unsupported"}
ARCH_TOY, ARCH_GPS, ARCH_DEPTH, ARCH_RGBD, ARCH_SERX50, ARCH_SERX101 = 0, 1, 2, 3, 4, 5
A8_SHARDED, A8_ALLREAD, A8_AUTO = 0, 1, 2


class DdppoError(RuntimeError):
    def __init__(self, fn, code, msg=""):
        super().__init__(f"{fn} -> {STATUS.get(code, code)} ({code}) {msg}")
        self.code = code


class ModelDesc(ctypes.Structure):
    _fields_ = [("arch", c_i32), ("hidden", c_i32), ("num_actions", c_i32), ("reserved", c_i32 * 5)]


class TensorInfo(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 48), ("offset", c_i64), ("numel", c_i64), ("ndim", c_i32),
                ("fan_in", c_i32), ("shape", c_i64 * 4)]


class Batch(ctypes.Structure):
    _fields_ = [("goal", c_vp), ("prev_action", c_vp), ("mask", c_vp), ("h0", c_vp), ("len", c_vp),
                ("env_idx", c_vp), ("E", c_i32), ("T", c_i32), ("ld", c_i32), ("B", c_i32), ("T_run", c_i32),
                ("n_valid", c_i32), ("obs", c_vp), ("c0", c_vp), ("obs_rgb", c_vp), ("dgoal", c_vp),
                ("flags", c_i32), ("reserved_flags", c_i32)]


class LossInputs(ctypes.Structure):
    _fields_ = [("action", c_vp), ("logp_old", c_vp), ("value_old", c_vp), ("ret", c_vp), ("adv", c_vp)]


class LossCfg(ctypes.Structure):
    _fields_ = [("clip_eps", c_float), ("vclip_eps", c_float), ("c_v", c_float), ("c_e", c_float),
                ("use_value_clip", c_i32), ("normalize_adv", c_i32)]


class AdamCfg(ctypes.Structure):
    _fields_ = [("lr", c_float), ("beta1", c_float), ("beta2", c_float), ("eps", c_float),
                ("max_grad_norm", c_float), ("step", c_i32)]


class PreemptCfg(ctypes.Structure):
    _fields_ = [("p_percent", c_i32), ("T", c_i32), ("min_steps", c_i32), ("other_workers", c_i32)]


class Rollout(ctypes.Structure):
    _fields_ = [("rew", c_vp), ("val", c_vp), ("done", c_vp), ("len", c_vp), ("goal", c_vp), ("prev_action", c_vp),
                ("mask", c_vp), ("h0", c_vp), ("action", c_vp), ("logp_old", c_vp), ("perms", c_vp),
                ("host_len", c_vp), ("host_perms", c_vp), ("E", c_i32), ("T", c_i32), ("ld", c_i32),
                ("obs", c_vp), ("c0", c_vp), ("obs_rgb", c_vp)]


class LearnerCfg(ctypes.Structure):
    _fields_ = [("gamma", c_float), ("tau", c_float), ("adv_eps", c_float), ("normalize_adv", c_i32),
                ("epochs", c_i32), ("minibatches", c_i32), ("loss", LossCfg), ("adam", AdamCfg),
                ("freeze_mask", c_vp), ("freeze_encoder", c_i32), ("reserved", c_i32)]


class ActBatch(ctypes.Structure):
    _fields_ = [("goal", c_vp), ("prev_action", c_vp), ("mask", c_vp), ("obs", c_vp), ("obs_rgb", c_vp),
                ("E", c_i32), ("T", c_i32), ("ld", c_i32), ("t", c_i32), ("h_in", c_vp), ("c_in", c_vp),
                ("h_out", c_vp), ("c_out", c_vp), ("seed", ctypes.c_uint64), ("counter", c_i64),
                ("greedy", c_i32), ("reserved", c_i32)]


P_ = ctypes.POINTER
_SIGS = {
    "ddppo_abi_version": (c_int, []),
    "ddppo_status_string": (ctypes.c_char_p, [c_int]),
    "ddppo_get_unique_id": (c_int, [c_vp]),
    "ddppo_ctx_create": (c_int, [c_int, c_int, c_vp, c_int, P_(c_vp)]),
    "ddppo_ctx_destroy": (c_int, [c_vp]),
    "ddppo_last_error": (ctypes.c_char_p, [c_vp]),
    "ddppo_check": (c_int, [c_vp, c_vp]),
    "ddppo_gae": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_int, c_int, c_int, c_float, c_float, c_vp, c_vp, c_vp,
                          c_vp]),
    "ddppo_adv_norm": (c_int, [c_vp, c_vp, c_float, c_vp, c_vp]),
    "ddppo_model_param_count": (c_int, [P_(ModelDesc), P_(c_i64)]),
    "ddppo_model_param_layout": (c_int, [P_(ModelDesc), c_vp, c_int, P_(c_int)]),
    "ddppo_workspace_size": (c_int, [P_(ModelDesc), c_int, c_int, P_(c_size)]),
    "ddppo_policy_fwd": (c_int, [c_vp, P_(ModelDesc), c_vp, P_(Batch), c_vp, c_vp, c_vp, c_size, c_vp]),
    "ddppo_policy_bwd": (c_int, [c_vp, P_(ModelDesc), c_vp, P_(Batch), c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "ddppo_ppo_loss_grad": (c_int, [c_vp, c_vp, c_vp, P_(Batch), P_(LossInputs), c_vp, P_(LossCfg), c_vp, c_vp,
                                    c_vp, c_vp]),
    "ddppo_grad_allreduce_step": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, P_(AdamCfg), c_vp, c_vp]),
    "ddppo_preempt_threshold": (c_int, [P_(PreemptCfg), c_int, P_(c_int), P_(c_int)]),
    "ddppo_preempt_decide": (c_int, [P_(PreemptCfg), c_int, c_int, c_int, P_(c_int)]),
    "ddppo_preempt_poll": (c_int, [c_vp, c_int, c_int, c_int, P_(PreemptCfg), P_(c_int), P_(c_int), P_(c_int)]),
    "ddppo_allreduce_counts": (c_int, [c_vp, c_vp, c_int]),
    "ddppo_learner_workspace_size": (c_int, [P_(ModelDesc), c_int, c_int, c_int, c_int, c_int, P_(c_size)]),
    "ddppo_learner_step": (c_int, [c_vp, P_(ModelDesc), P_(Rollout), P_(LearnerCfg), c_vp, c_vp, c_vp, c_vp, c_vp,
                                   c_vp, c_vp, c_size, P_(c_i32), c_vp]),
    "ddppo_profile_enable": (c_int, [c_vp, c_int]),
    "ddppo_profile_read": (c_int, [c_vp, c_vp, c_vp, c_int]),
    "ddppo_profile_flops": (c_int, [c_vp, c_vp, c_int]),
    "ddppo_profile_smem_bytes": (c_int, [c_vp, c_vp, c_int]),
    "ddppo_rollout_steps": (c_int, [c_vp, c_int, c_int, c_vp]),
    "ddppo_debug_gemm_bf16": (c_int, [c_vp, c_vp, c_i64, c_i64, c_vp, c_i64, c_i64, c_vp, c_i64, c_int, c_int, c_int,
                                      c_int, c_vp, c_int, c_vp]),
    "ddppo_debug_conv2d": (c_int, [c_vp, c_vp, c_vp, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_vp,
                                   c_vp, c_vp, c_vp, c_vp, ctypes.c_size_t, c_vp, c_vp]),
    "ddppo_debug_groupnorm": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_int, c_int, c_int, c_int, c_vp, c_vp, c_vp,
                                      c_vp, c_vp, c_vp, c_vp, c_vp]),
    "ddppo_debug_depth_decisions": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "ddppo_learner_register": (c_int, [c_vp, c_vp, ctypes.c_size_t]),
    "ddppo_set_graphs": (c_int, [c_vp, c_int]),
    "ddppo_set_a8_mode": (c_int, [c_vp, c_int]),
    "ddppo_set_conv_engine": (c_int, [c_vp, c_int]),
    "ddppo_set_fwd_planes": (c_int, [c_vp, c_int]),
    "ddppo_act_workspace_size": (c_int, [P_(ModelDesc), c_int, P_(c_size)]),
    "ddppo_policy_act": (c_int, [c_vp, P_(ModelDesc), c_vp, P_(ActBatch), c_vp, c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "ddppo_reinit_critic": (c_int, [c_vp, P_(ModelDesc), c_vp, c_vp, c_vp, ctypes.c_uint64, c_vp]),
    "ddppo_layout_hash": (c_int, [P_(ModelDesc), c_int, c_int, c_int, c_int, c_int, P_(ctypes.c_uint64)]),
    "ddppo_layout_check": (c_int, [c_vp, P_(ModelDesc), c_int, c_int, c_int, c_int, c_int]),
    "ddppo_debug_peer_a8": (c_int, [c_vp, c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_i64, P_(AdamCfg), c_vp, c_vp,
                                    c_size, P_(c_size), c_vp]),
    "ddppo_debug_peer_counts": (c_int, [c_vp, c_int, c_vp, c_int, c_vp, c_vp, c_size, P_(c_size)]),
    "ddppo_debug_maxpool": (c_int, [c_vp, c_vp, c_int, c_int, c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp]),
}
KERNEL_FAMILIES = ("gae", "adv_norm", "net_fwd", "head", "loss", "net_bwd", "wgrad", "allreduce", "adam", "other",
                   "conv", "rnn", "gn")
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTS = tuple(_SIGS)


def check(fn, code, ctx=None):
    if code != 0:
        msg = lib.ddppo_last_error(ctx).decode() if ctx else ""
        raise DdppoError(fn, code, msg)


def ptr(t):
    """Device (or host) address of a torch tensor / numpy array, or None."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def dptr(t, dtype=None):
    """Device address of a contiguous CUDA torch tensor of `dtype` (loud failure otherwise)."""
    if t is None:
        return None
    if not getattr(t, "is_cuda", False):
        raise TypeError("expected a CUDA tensor (no CPU path exists)")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    if dtype is not None and str(t.dtype) != "torch." + dtype:
        raise TypeError(f"expected torch.{dtype}, got {t.dtype}")
    return t.data_ptr()


def f32(t):
    return dptr(t, "float32")


def f64(t):
    return dptr(t, "float64")


def i32(t):
    return dptr(t, "int32")


def u8(t):
    return dptr(t, "uint8")
