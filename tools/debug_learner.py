import numpy as np, torch, synth
import paper_1911_00357_b200 as dd
from oracle import learner as olearner
from paper_1911_00357_b200.learner import Learner
ctx = dd.Context(0, 1)
E, T = 2, 16
desc = dd.model_desc("gps"); lay = dd.param_layout(desc); P = dd.param_count(desc)
p0 = synth.init_params([(off, int(np.prod(s)), fan) for _, off, s, fan in lay], P, 0)
for lengths in ([16, 16], [16, 9]):
    lrn = Learner(ctx, "gps", E, T, epochs=1, minibatches=1, params=p0)
    ro = synth.rollout(E, T, 0, length=lengths, hidden=512)
    pm = synth.perms(0, 0, 1, E)
    lrn.load_rollout(ro, pm)
    stats = lrn.step().cpu().numpy()
    tr = []
    po, _, _, _, info = olearner.learner_step("gps", p0, np.zeros(P), np.zeros(P), 0, [ro], [pm], dict(epochs=1, minibatches=1), trace=tr)
    print("lengths", lengths, "perm", pm, "host_perms", lrn.host_perms, "host_len", lrn.host_len)
    print("gpu stats", stats[0]); print("ora stats", info["mb_stats"][0])
    lg = lrn.ws[128:128 + 2 * 16 * 4].view(2, 16, 4).cpu().numpy()
    print("gpu logits", lg[0, :2], lg[1, :2]); print("ora logits", tr[0]["logits"][0, :2], tr[0]["logits"][1, :2])
    print("dev len", lrn.dev["length"].cpu().numpy(), "perms dev", lrn.perms.cpu().numpy())
