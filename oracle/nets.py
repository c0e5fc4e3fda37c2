"""Textbook layer definitions with manual backward passes (step a5/a7).

Test infrastructure only.  NumPy float64.  Conventions (Z21):
PyTorch's Linear (y = x W^T + b), Embedding, GRU (gate rows r, z, n;
n = tanh(W_in x + b_in + r * (W_hn h + b_hn))) and LSTM (gate rows i, f, g, o,
two bias vectors).  The recurrent state is multiplied by mask_t before step
t (episode reset, "start-token in the case of the first action");
no gradient flows into h0/c0 (they are inputs of the rollout).
"""
import numpy as np


def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


# ---------------------------------------------------------------- Linear
def linear_fwd(x, W, b):
    return x @ W.T + b


def linear_bwd(x, W, dy):
    """returns dx, dW, db for y = x W^T + b (x: [..., I], dy: [..., O])."""
    x2 = x.reshape(-1, x.shape[-1])
    d2 = dy.reshape(-1, dy.shape[-1])
    return (dy @ W), d2.T @ x2, d2.sum(axis=0)


# ---------------------------------------------------------------- Embedding
def embedding_fwd(idx, table):
    return table[np.asarray(idx, dtype=np.int64)]


def embedding_bwd(idx, dy, n_rows):
    d = np.zeros((n_rows, dy.shape[-1]))
    np.add.at(d, np.asarray(idx, dtype=np.int64).reshape(-1), dy.reshape(-1, dy.shape[-1]))
    return d


# ---------------------------------------------------------------- GRU
def gru_seq_fwd(x, mask, h0, W_ih, W_hh, b_ih, b_hh):
    """x [B][T][I], mask [B][T], h0 [B][H] -> h [B][T][H], cache."""
    B, T, _ = x.shape
    H = W_hh.shape[1]
    h = np.zeros((B, T, H))
    cache = {"x": x, "mask": mask, "h_in": np.zeros((B, T, H)), "r": np.zeros((B, T, H)),
             "z": np.zeros((B, T, H)), "n": np.zeros((B, T, H)), "ghn": np.zeros((B, T, H))}
    hp = h0
    for t in range(T):
        h_in = mask[:, t:t + 1] * hp
        gi = x[:, t] @ W_ih.T + b_ih
        gh = h_in @ W_hh.T + b_hh
        r = sigmoid(gi[:, :H] + gh[:, :H])
        z = sigmoid(gi[:, H:2 * H] + gh[:, H:2 * H])
        ghn = gh[:, 2 * H:]
        n = np.tanh(gi[:, 2 * H:] + r * ghn)
        hn = (1.0 - z) * n + z * h_in
        for k, val in (("h_in", h_in), ("r", r), ("z", z), ("n", n), ("ghn", ghn)):
            cache[k][:, t] = val
        h[:, t] = hn
        hp = hn
    return h, cache


def gru_seq_bwd(dh_out, cache, W_ih, W_hh):
    """BPTT.  dh_out [B][T][H] = dL/dh_t from above.  Returns dx, dW_ih, dW_hh, db_ih, db_hh."""
    x, mask = cache["x"], cache["mask"]
    B, T, H = dh_out.shape
    dx = np.zeros_like(x)
    dW_ih = np.zeros_like(W_ih)
    dW_hh = np.zeros_like(W_hh)
    db_ih = np.zeros(3 * H)
    db_hh = np.zeros(3 * H)
    carry = np.zeros((B, H))
    for t in range(T - 1, -1, -1):
        r, z, n, ghn, h_in = (cache[k][:, t] for k in ("r", "z", "n", "ghn", "h_in"))
        dh = dh_out[:, t] + carry
        dn = dh * (1.0 - z)
        dz = dh * (h_in - n)
        dn_pre = dn * (1.0 - n * n)
        dr = dn_pre * ghn
        dr_pre = dr * r * (1.0 - r)
        dz_pre = dz * z * (1.0 - z)
        dgi = np.concatenate([dr_pre, dz_pre, dn_pre], axis=1)
        dgh = np.concatenate([dr_pre, dz_pre, dn_pre * r], axis=1)
        dW_ih += dgi.T @ x[:, t]
        dW_hh += dgh.T @ h_in
        db_ih += dgi.sum(axis=0)
        db_hh += dgh.sum(axis=0)
        dx[:, t] = dgi @ W_ih
        dh_in = dh * z + dgh @ W_hh
        carry = mask[:, t:t + 1] * dh_in
    return dx, dW_ih, dW_hh, db_ih, db_hh


# ---------------------------------------------------------------- LSTM
def lstm_seq_fwd(x, mask, h0, c0, W_ih, W_hh, b_ih, b_hh):
    """x [B][T][I] -> h [B][T][H]; gates i, f, g, o (PyTorch order)."""
    B, T, _ = x.shape
    H = W_hh.shape[1]
    h = np.zeros((B, T, H))
    keys = ("h_in", "c_in", "i", "f", "g", "o", "c")
    cache = {k: np.zeros((B, T, H)) for k in keys}
    cache["x"], cache["mask"] = x, mask
    hp, cp = h0, c0
    for t in range(T):
        h_in = mask[:, t:t + 1] * hp
        c_in = mask[:, t:t + 1] * cp
        g_all = x[:, t] @ W_ih.T + b_ih + h_in @ W_hh.T + b_hh
        i = sigmoid(g_all[:, :H])
        f = sigmoid(g_all[:, H:2 * H])
        g = np.tanh(g_all[:, 2 * H:3 * H])
        o = sigmoid(g_all[:, 3 * H:])
        c = f * c_in + i * g
        hn = o * np.tanh(c)
        for k, val in zip(keys, (h_in, c_in, i, f, g, o, c)):
            cache[k][:, t] = val
        h[:, t] = hn
        hp, cp = hn, c
    return h, cache


def lstm_seq_bwd(dh_out, cache, W_ih, W_hh):
    x, mask = cache["x"], cache["mask"]
    B, T, H = dh_out.shape
    dx = np.zeros_like(x)
    dW_ih = np.zeros_like(W_ih)
    dW_hh = np.zeros_like(W_hh)
    db = np.zeros(4 * H)
    dh_carry = np.zeros((B, H))
    dc_carry = np.zeros((B, H))
    for t in range(T - 1, -1, -1):
        h_in, c_in, i, f, g, o, c = (cache[k][:, t] for k in ("h_in", "c_in", "i", "f", "g", "o", "c"))
        dh = dh_out[:, t] + dh_carry
        tc = np.tanh(c)
        do = dh * tc
        dc = dh * o * (1.0 - tc * tc) + dc_carry
        di = dc * g
        dg = dc * i
        df = dc * c_in
        dc_in = dc * f
        dgates = np.concatenate([di * i * (1 - i), df * f * (1 - f), dg * (1 - g * g), do * o * (1 - o)], axis=1)
        dW_ih += dgates.T @ x[:, t]
        dW_hh += dgates.T @ h_in
        db += dgates.sum(axis=0)
        dx[:, t] = dgates @ W_ih
        dh_in = dgates @ W_hh
        dh_carry = mask[:, t:t + 1] * dh_in
        dc_carry = mask[:, t:t + 1] * dc_in
    return dx, dW_ih, dW_hh, db.copy(), db.copy()
