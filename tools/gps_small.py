import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch, synth
import paper_1911_00357_b200 as dd
from paper_1911_00357_b200.learner import Learner
T = int(sys.argv[1]) if len(sys.argv) > 1 else 4
ctx = dd.Context(0, 1)
c = dict(synth.CONFIGS["gps"]); c["T"] = T
desc = dd.model_desc(c["arch"]); lay = dd.param_layout(desc); P = dd.param_count(desc)
p0 = synth.init_params([(off, int(np.prod(s)), fan) for _, off, s, fan in lay], P, 0)
lrn = Learner(ctx, c["arch"], c["E"], c["T"], c["epochs"], c["minibatches"], params=p0, normalize_adv=True)
ro = synth.rollout(c["E"], c["T"], 0, hidden=desc.hidden)
pm = synth.perms(0, 0, c["epochs"], c["E"])
lrn.load_rollout(ro, pm)
print("loaded", flush=True)
lrn.step()
torch.cuda.synchronize(); ctx.check()
print("ok", flush=True)
