"""Actor-critic assemblies and their flat-parameter layouts (steps a5, a7).

Test infrastructure only.  The layouts are re-implemented here from the
documented order in include/ddppo.h / DESIGN.md ("Flat parameter layout"),
not from the CUDA code.  Rule: tensors are laid out in the listed order,
row-major, each starting at an offset rounded up to a multiple of 4 floats
(no padding happens for the shipped configs).

Architectures (BASELINE.json configs; readings Z17-Z22):
  toy  (configs[0]): goal [d, cos, sin] -> Linear(3,64) -> tanh
                     -> Linear(64, A+1)   (A = 4 actions; +1 value)
  gps  (configs[1]): goal -> Linear(3,32) (linear);
                     prev action -> Embedding(A+1, 32), start token = A;
                     x = [goal_emb, act_emb] (Z22 order) -> GRU(64, 512)
                     -> Linear(512, A+1) ("fully connected layer,
                     resulting in a soft-max distribution ... and an estimate
                     of the value function").
  depth (configs[2]): depth [1][64][64] -> half-width ResNet18 (convnets.py)
                     -> 128x2x2 -> flatten (c, h, w order) -> Linear(512, 512) + ReLU
                     (Z17, Z20); x = [visual 512, goal_fc 32, act_emb 32]
                     -> LSTM(576, 512) (PyTorch i, f, g, o) -> Linear(512, A+1).
  serx50 / serx101 (NEXT-3, P:L212 / P:L313-318 / P:L582): the RGB-D agent with the half-width
                     SE-ResNeXt50 / 101 encoder (convnets.serx50h_*; reading R9), same policy.
  rgbd (configs[3]): RGB-D [4][256][256] (RGB in [0, 255] normalised channel-wise) ->
                     2x2 avg-pool -> half-width ResNet50 (convnets.py) -> 128x4x4 -> flatten ->
                     Linear(2048, 512) + ReLU; x = [visual, goal_fc, act_emb] -> 2-layer LSTM-512
                     (layer 2 reads layer 1's h) -> Linear(512, A+1).  h0 / c0 are
                     [B][2*512] (layer-major).
fan_in > 0: U(+-1/sqrt(fan_in)) default init; fan_in == 0: ones (GN gamma);
fan_in < 0: zeros (GN beta).
"""
import numpy as np

from . import convnets, nets

NUM_ACTIONS = 4


def layout(arch, hidden=512, num_actions=NUM_ACTIONS):
    """Ordered [(name, shape, fan_in)]."""
    A1 = num_actions + 1
    if arch == "toy":
        h = 64
        return [("fc1.weight", (h, 3), 3), ("fc1.bias", (h,), 3),
                ("head.weight", (A1, h), h), ("head.bias", (A1,), h)]
    if arch == "gps":
        H, G = hidden, 3 * hidden
        return [("goal_fc.weight", (32, 3), 3), ("goal_fc.bias", (32,), 3),
                ("act_embed.weight", (A1, 32), 1),
                ("rnn.weight_ih", (G, 64), H), ("rnn.weight_hh", (G, H), H),
                ("rnn.bias_ih", (G,), H), ("rnn.bias_hh", (G,), H),
                ("head.weight", (A1, H), H), ("head.bias", (A1,), H)]
    if arch == "depth":
        H, G = hidden, 4 * hidden
        out = []
        for name, kind, shape, _, _ in convnets.resnet18h_spec(1):
            if kind == "conv":
                out.append((name + ".weight", shape, shape[1] * shape[2] * shape[3]))
            else:
                out += [(name + ".weight", shape, 0), (name + ".bias", shape, -1)]
        return out + [("visual_fc.weight", (512, 512), 512), ("visual_fc.bias", (512,), 512),
                      ("goal_fc.weight", (32, 3), 3), ("goal_fc.bias", (32,), 3),
                      ("act_embed.weight", (A1, 32), 1),
                      ("rnn.weight_ih", (G, 576), H), ("rnn.weight_hh", (G, H), H),
                      ("rnn.bias_ih", (G,), H), ("rnn.bias_hh", (G,), H),
                      ("head.weight", (A1, H), H), ("head.bias", (A1,), H)]
    if arch in ("rgbd", "serx50", "serx101"):
        H, G = hidden, 4 * hidden
        out = []
        spec = (convnets.resnet50h_spec(4) if arch == "rgbd" else
                convnets.serx50h_spec(4, convnets.R101_BLOCKS if arch == "serx101" else convnets.R50_BLOCKS))
        for name, kind, shape, _, _ in spec:
            if kind in ("conv", "gconv"):
                out.append((name + ".weight", shape, shape[1] * shape[2] * shape[3]))
            elif kind == "fc":  # SE linear layer: torch's default init U(+-1/sqrt(fan_in)), weight and bias
                out += [(name + ".weight", shape, shape[1]), (name + ".bias", shape[:1], shape[1])]
            else:
                out += [(name + ".weight", shape, 0), (name + ".bias", shape, -1)]
        out += [("visual_fc.weight", (512, 2048), 2048), ("visual_fc.bias", (512,), 2048),
                ("goal_fc.weight", (32, 3), 3), ("goal_fc.bias", (32,), 3),
                ("act_embed.weight", (A1, 32), 1)]
        for layer, nin in ((0, 576), (1, H)):
            out += [(f"rnn.weight_ih_l{layer}", (G, nin), H), (f"rnn.weight_hh_l{layer}", (G, H), H),
                    (f"rnn.bias_ih_l{layer}", (G,), H), (f"rnn.bias_hh_l{layer}", (G,), H)]
        return out + [("head.weight", (A1, H), H), ("head.bias", (A1,), H)]
    raise ValueError(arch)


def _serx_blocks(arch):
    return convnets.R101_BLOCKS if arch == "serx101" else convnets.R50_BLOCKS


def offsets(arch, **kw):
    out, off = {}, 0
    for name, shape, _ in layout(arch, **kw):
        off = (off + 3) // 4 * 4
        n = int(np.prod(shape))
        out[name] = (off, shape)
        off += n
    return out, off


def unpack(arch, flat, **kw):
    offs, _ = offsets(arch, **kw)
    flat = np.asarray(flat, dtype=np.float64)
    return {k: flat[o:o + int(np.prod(s))].reshape(s) for k, (o, s) in offs.items()}


def pack(arch, tensors, **kw):
    """Tensors missing from `tensors` (a frozen encoder's, NEXT-4) are packed as zeros."""
    offs, P = offsets(arch, **kw)
    flat = np.zeros(P)
    for k, (o, s) in offs.items():
        if k in tensors:
            flat[o:o + int(np.prod(s))] = np.asarray(tensors[k], dtype=np.float64).reshape(-1)
    return flat


# ---------------------------------------------------------------- forward / backward
def forward(arch, flat, batch, **kw):
    """batch: goal [B][T][3], prev_action [B][T], mask [B][T], h0 [B][H].

    Returns logits [B][T][A], values [B][T], cache.
    """
    p = unpack(arch, flat, **kw)
    goal = np.asarray(batch["goal"], dtype=np.float64)
    if arch == "toy":
        pre = nets.linear_fwd(goal, p["fc1.weight"], p["fc1.bias"])
        h = np.tanh(pre)
        out = nets.linear_fwd(h, p["head.weight"], p["head.bias"])
        cache = {"goal": goal, "h": h}
    elif arch == "gps":
        ge = nets.linear_fwd(goal, p["goal_fc.weight"], p["goal_fc.bias"])
        ae = nets.embedding_fwd(batch["prev_action"], p["act_embed.weight"])
        x = np.concatenate([ge, ae], axis=-1)
        h, rc = nets.gru_seq_fwd(x, np.asarray(batch["mask"], dtype=np.float64),
                                 np.asarray(batch["h0"], dtype=np.float64),
                                 p["rnn.weight_ih"], p["rnn.weight_hh"], p["rnn.bias_ih"], p["rnn.bias_hh"])
        out = nets.linear_fwd(h, p["head.weight"], p["head.bias"])
        cache = {"goal": goal, "prev_action": np.asarray(batch["prev_action"]), "h": h, "rnn": rc}
    elif arch == "depth":
        obs = np.asarray(batch["obs"], dtype=np.float64)  # [B][T][1][H][W]
        B, T = obs.shape[:2]
        feat, ec = convnets.resnet18h_fwd(obs.reshape((B * T,) + obs.shape[2:]), p)
        flat_f = feat.reshape(B, T, -1)  # (c, h, w) order
        vpre = nets.linear_fwd(flat_f, p["visual_fc.weight"], p["visual_fc.bias"])
        vis = np.maximum(vpre, 0.0)
        ge = nets.linear_fwd(goal, p["goal_fc.weight"], p["goal_fc.bias"])
        ae = nets.embedding_fwd(batch["prev_action"], p["act_embed.weight"])
        x = np.concatenate([vis, ge, ae], axis=-1)
        H = p["rnn.weight_hh"].shape[1]
        c0 = np.asarray(batch.get("c0", np.zeros((B, H))), dtype=np.float64)
        h, rc = nets.lstm_seq_fwd(x, np.asarray(batch["mask"], dtype=np.float64),
                                  np.asarray(batch["h0"], dtype=np.float64), c0,
                                  p["rnn.weight_ih"], p["rnn.weight_hh"], p["rnn.bias_ih"], p["rnn.bias_hh"])
        out = nets.linear_fwd(h, p["head.weight"], p["head.bias"])
        cache = {"goal": goal, "prev_action": np.asarray(batch["prev_action"]), "h": h, "rnn": rc, "enc": ec,
                 "feat_shape": feat.shape, "flat": flat_f, "vis": vis}
    elif arch in ("rgbd", "serx50", "serx101"):
        obs = np.asarray(batch["obs"], dtype=np.float64)  # [B][T][4][256][256]
        B, T = obs.shape[:2]
        if arch == "rgbd":
            feat, ec = convnets.resnet50h_fwd(obs.reshape((B * T,) + obs.shape[2:]), p)
        else:
            feat, ec = convnets.serx50h_fwd(obs.reshape((B * T,) + obs.shape[2:]), p, _serx_blocks(arch))
        flat_f = feat.reshape(B, T, -1)  # (c, h, w) order, 2048
        vis = np.maximum(nets.linear_fwd(flat_f, p["visual_fc.weight"], p["visual_fc.bias"]), 0.0)
        ge = nets.linear_fwd(goal, p["goal_fc.weight"], p["goal_fc.bias"])
        ae = nets.embedding_fwd(batch["prev_action"], p["act_embed.weight"])
        H = p["rnn.weight_hh_l0"].shape[1]
        mask = np.asarray(batch["mask"], dtype=np.float64)
        h0 = np.asarray(batch["h0"], dtype=np.float64).reshape(B, 2, H)
        c0 = np.asarray(batch["c0"], dtype=np.float64).reshape(B, 2, H)
        x = np.concatenate([vis, ge, ae], axis=-1)
        rcs = []
        for layer in range(2):
            x, rc = nets.lstm_seq_fwd(x, mask, h0[:, layer], c0[:, layer], p[f"rnn.weight_ih_l{layer}"],
                                      p[f"rnn.weight_hh_l{layer}"], p[f"rnn.bias_ih_l{layer}"],
                                      p[f"rnn.bias_hh_l{layer}"])
            rcs.append(rc)
        h = x
        out = nets.linear_fwd(h, p["head.weight"], p["head.bias"])
        cache = {"goal": goal, "prev_action": np.asarray(batch["prev_action"]), "h": h, "rnn": rcs, "enc": ec,
                 "feat_shape": feat.shape, "flat": flat_f, "vis": vis}
    else:
        raise ValueError(arch)
    return out[..., :-1], out[..., -1], cache


def backward(arch, flat, cache, dlogits, dvalues, freeze_encoder=False, extra=None, **kw):
    """dlogits [B][T][A], dvalues [B][T] -> flat gradient [P].

    Transfer mechanics (NEXT-4), visual agents: freeze_encoder -- the visual encoder
    (enc.* tensors) is frozen, so the backward stops at the visual FC and the encoder's gradient is 0;
    extra (a dict) receives "dgoal" [B][T][3] = dL/d(goal input), the gradient a planner gets
    through a frozen controller."""
    p = unpack(arch, flat, **kw)
    dout = np.concatenate([dlogits, dvalues[..., None]], axis=-1)
    g = {}
    if arch == "toy":
        dh, g["head.weight"], g["head.bias"] = nets.linear_bwd(cache["h"], p["head.weight"], dout)
        dpre = dh * (1.0 - cache["h"] ** 2)
        _, g["fc1.weight"], g["fc1.bias"] = nets.linear_bwd(cache["goal"], p["fc1.weight"], dpre)
    elif arch == "gps":
        dh, g["head.weight"], g["head.bias"] = nets.linear_bwd(cache["h"], p["head.weight"], dout)
        dx, g["rnn.weight_ih"], g["rnn.weight_hh"], g["rnn.bias_ih"], g["rnn.bias_hh"] = \
            nets.gru_seq_bwd(dh, cache["rnn"], p["rnn.weight_ih"], p["rnn.weight_hh"])
        dge, dae = dx[..., :32], dx[..., 32:]
        _, g["goal_fc.weight"], g["goal_fc.bias"] = nets.linear_bwd(cache["goal"], p["goal_fc.weight"], dge)
        g["act_embed.weight"] = nets.embedding_bwd(cache["prev_action"], dae, p["act_embed.weight"].shape[0])
    elif arch == "depth":
        dh, g["head.weight"], g["head.bias"] = nets.linear_bwd(cache["h"], p["head.weight"], dout)
        dx, g["rnn.weight_ih"], g["rnn.weight_hh"], g["rnn.bias_ih"], g["rnn.bias_hh"] = \
            nets.lstm_seq_bwd(dh, cache["rnn"], p["rnn.weight_ih"], p["rnn.weight_hh"])
        dvis, dge, dae = dx[..., :512], dx[..., 512:544], dx[..., 544:]
        dgoal, g["goal_fc.weight"], g["goal_fc.bias"] = nets.linear_bwd(cache["goal"], p["goal_fc.weight"], dge)
        if extra is not None:
            extra["dgoal"] = dgoal
        g["act_embed.weight"] = nets.embedding_bwd(cache["prev_action"], dae, p["act_embed.weight"].shape[0])
        dvpre = dvis * (cache["vis"] > 0)
        dflat, g["visual_fc.weight"], g["visual_fc.bias"] = nets.linear_bwd(cache["flat"], p["visual_fc.weight"],
                                                                            dvpre)
        if not freeze_encoder:
            convnets.resnet18h_bwd(dflat.reshape(cache["feat_shape"]), p, cache["enc"], g)
    elif arch in ("rgbd", "serx50", "serx101"):
        dh, g["head.weight"], g["head.bias"] = nets.linear_bwd(cache["h"], p["head.weight"], dout)
        for layer in (1, 0):
            dh, g[f"rnn.weight_ih_l{layer}"], g[f"rnn.weight_hh_l{layer}"], g[f"rnn.bias_ih_l{layer}"], \
                g[f"rnn.bias_hh_l{layer}"] = nets.lstm_seq_bwd(dh, cache["rnn"][layer], p[f"rnn.weight_ih_l{layer}"],
                                                               p[f"rnn.weight_hh_l{layer}"])
        dx = dh
        dvis, dge, dae = dx[..., :512], dx[..., 512:544], dx[..., 544:]
        dgoal, g["goal_fc.weight"], g["goal_fc.bias"] = nets.linear_bwd(cache["goal"], p["goal_fc.weight"], dge)
        if extra is not None:
            extra["dgoal"] = dgoal
        g["act_embed.weight"] = nets.embedding_bwd(cache["prev_action"], dae, p["act_embed.weight"].shape[0])
        dvpre = dvis * (cache["vis"] > 0)
        dflat, g["visual_fc.weight"], g["visual_fc.bias"] = nets.linear_bwd(cache["flat"], p["visual_fc.weight"],
                                                                            dvpre)
        if not freeze_encoder:
            if arch == "rgbd":
                convnets.resnet50h_bwd(dflat.reshape(cache["feat_shape"]), p, cache["enc"], g)
            else:
                convnets.serx50h_bwd(dflat.reshape(cache["feat_shape"]), p, cache["enc"], g, _serx_blocks(arch))
    else:
        raise ValueError(arch)
    return pack(arch, g, **kw)
