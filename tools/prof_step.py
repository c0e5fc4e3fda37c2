"""One GPS learner step (after warm-up) for ncu captures: python tools/prof_step.py [steps] [config]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_1911_00357_b200 as dd
from paper_1911_00357_b200.learner import Learner
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = sys.argv[2] if len(sys.argv) > 2 else "gps"
ctx = dd.Context(0, 1)
c = synth.CONFIGS[cfg]
desc = dd.model_desc(c["arch"]); lay = dd.param_layout(desc); P = dd.param_count(desc)
p0 = synth.init_params([(off, int(np.prod(s)), fan) for _, off, s, fan in lay], P, 0)
lrn = Learner(ctx, c["arch"], c["E"], c["T"], c["epochs"], c["minibatches"], params=p0, normalize_adv=True)
ro = synth.rollout(c["E"], c["T"], 0, hidden=desc.hidden, obs_shape=c.get("obs"), rnn_layers=c.get("rnn_layers", 1))
pm = synth.perms(0, 0, c["epochs"], c["E"])
lrn.load_rollout(ro, pm)
for i in range(steps):
    lrn.step()
torch.cuda.synchronize(); ctx.check()
print("ok", lrn.stats[0].tolist())
