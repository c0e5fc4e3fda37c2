import numpy as np, torch, synth
import paper_1911_00357_b200 as dd
from oracle import models
ctx = dd.Context(0, 1)
E, T, B = 2, 16, 2
desc = dd.model_desc("gps"); lay = dd.param_layout(desc); P = dd.param_count(desc)
params = synth.init_params([(off, int(np.prod(s)), fan) for _, off, s, fan in lay], P, 0)
ro = synth.rollout(E, T, 0, hidden=512)
env_idx = np.arange(B, dtype=np.int32)
T_run = T
cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
keep = [cu(ro[k]) for k in ("goal", "prev_action", "mask", "h0", "length")] + [cu(env_idx)]
batch = dd.make_batch(*keep, E, T, ro["ld"], B, T_run, B * T)
ws = torch.zeros(dd.workspace_size(desc, B, T_run) // 4 + 64, device="cuda")
lg = torch.zeros((B, T_run, 4), device="cuda"); vl = torch.zeros((B, T_run), device="cuda")
pg = cu(params)
dd.ddppo_policy_fwd(ctx, desc, pg, batch, lg, vl, ws)
torch.cuda.synchronize()
ob = {"goal": ro["goal"][env_idx, :T_run], "prev_action": ro["prev_action"][env_idx, :T_run], "mask": ro["mask"][env_idx, :T_run], "h0": ro["h0"][env_idx]}
lo, vo, cache = models.forward("gps", params, ob)
print("gpu logits", lg.cpu().numpy()[0, :4]); print("ora logits", lo[0, :4])
S = B * T_run
import ctypes
# inspect workspace pieces: X then GI then Hs
X = ws[:S * 64].view(S, 64).cpu().numpy()
p = models.unpack("gps", params)
ge = ob["goal"] @ p["goal_fc.weight"].T + p["goal_fc.bias"]
print("X gpu", X[1, :4], X[1, 32:36]); print("X ora", ge[0, 1, :4], p["act_embed.weight"][ob["prev_action"][0, 1]][:4])
off = ((S * 64 * 4 + 255) // 256 * 256) // 4
goff = off + ((S * 1536 * 4 + 255) // 256 * 256) // 4
Hs = ws[goff:goff + S * 512].view(B, T_run, 512).cpu().numpy()
print("H gpu", Hs[0, 0, :4], Hs[0, 5, 100:104]); print("H ora", cache["h"][0, 0, :4], cache["h"][0, 5, 100:104])
print("max |H| diff", np.abs(Hs - cache["h"]).max())
