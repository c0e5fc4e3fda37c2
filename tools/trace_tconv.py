"""Phase timing of the TMA conv kernel (debug build tools/libddppo_tctrace.so, -DDDPPO_TCONV_TRACE):
one eager Depth network forward + backward at the config's minibatch (B = 2, T = 128, F = 256 frames),
per launch: duration (first CTA entry -> last CTA exit), CTA start skew, and the median CTA's
prologue / wait / first-accumulator / epilogue-end / exit times (us, from that CTA's entry)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1911_00357_b200._lib as L
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libddppo_tctrace.so"))
for name, (res, args) in L._SIGS.items():
    f = getattr(lib, name); f.restype = res; f.argtypes = args
L.lib = lib
import paper_1911_00357_b200 as dd
dd.lib = lib
import torch, synth

cfg = sys.argv[1] if len(sys.argv) > 1 else "depth"
c = synth.CONFIGS[cfg]
ctx = dd.Context(0, 1)
desc = dd.model_desc(c["arch"], c["hidden"]); lay = dd.param_layout(desc); P = dd.param_count(desc)
p0 = synth.init_params([(off, int(np.prod(s)), fan) for _, off, s, fan in lay], P, 0)
ro = synth.rollout(c["E"], c["T"], 0, hidden=desc.hidden, obs_shape=c["obs"], rnn_layers=c.get("rnn_layers", 1))
E, T, B = c["E"], c["T"], c["E"] // c["minibatches"]
cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
env_idx = np.arange(B, dtype=np.int32)
rgbd = c["arch"] != "depth"
vo = {k: t.cuda() for k, t in dd.visual_obs(ro["obs"], rgbd).items()}
batch = dd.make_batch(cu(ro["goal"]), cu(ro["prev_action"]), cu(ro["mask"]), cu(ro["h0"]), cu(ro["length"]),
                      cu(env_idx), E, T, ro["ld"], B, T, B * T, obs=vo.get("obs"), c0=cu(ro["c0"]),
                      obs_rgb=vo.get("obs_rgb"))
ws = torch.zeros(dd.workspace_size(desc, B, T) // 4 + 64, device="cuda")
lg, vl = torch.zeros((B, T, 4), device="cuda"), torch.zeros((B, T), device="cuda")
pg = cu(p0)
grad = torch.zeros(P, device="cuda")
dl, dv = torch.full((B, T, 4), 1e-3, device="cuda"), torch.full((B, T), 1e-3, device="cuda")
for _ in range(3):
    dd.ddppo_policy_fwd(ctx, desc, pg, batch, lg, vl, ws)
    dd.ddppo_policy_bwd(ctx, desc, pg, batch, dl, dv, grad, ws)
torch.cuda.synchronize()
N = 1024
buf = (ctypes.c_ulonglong * (N * 160 * 8))()
meta = (ctypes.c_longlong * (N * 16))()
lib.ddppo_debug_tconv_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
lib.ddppo_debug_tconv_trace(ctypes.addressof(buf), ctypes.addressof(meta), N)
tr = np.array(buf, dtype=np.float64).reshape(N, 160, 8)
me = np.array(meta, dtype=np.int64).reshape(N, 16)
n = int(np.argmax(me[:, 4] == 0)) if (me[:, 4] == 0).any() else N  # launches recorded
per = n // 3  # the last of the three fwd + bwd passes
tot = 0.0
print(f"{'mode':>5} {'cs':>3} {'bn':>3} {'pl':>2} {'M':>7} {'N':>4} {'n_k':>4} {'kper':>4} {'work':>5} {'grid':>4} "
      f"{'slot':>4} {'spl':>3} | {'dur':>6} {'skew':>5} {'prol':>5} {'wait':>5} {'acc1':>6} {'epi':>6} {'exit':>6}  (us)")
for i in range(n - per, n):
    m = me[i]
    g = int(min(m[9], 160))
    t = tr[i, :g]
    t0 = t[:, 0]
    dur = (t[:, 6].max() - t0.min()) / 1e3
    tot += dur
    rel = lambda k: np.median(t[:, k] - t0) / 1e3  # noqa: E731
    names = {0: "FPROP", 1: "WGRAD", 2: "HALO"}
    print(f"{names.get(int(m[0]), m[0]):>5} {m[1]:3d} {m[2]:3d} {m[3]:2d} {m[4]:7d} {m[5]:4d} {m[6]:4d} {m[7]:4d} {m[8]:5d} "
          f"{m[9]:4d} {m[10]:4d} {m[11]:3d} | {dur:6.1f} {(t0.max() - t0.min()) / 1e3:5.1f} {rel(1):5.1f} {rel(2):5.1f} "
          f"{rel(4):6.1f} {rel(5):6.1f} {rel(6):6.1f}")
print(f"{per} launches per fwd+bwd, sum of durations {tot:.1f} us")
