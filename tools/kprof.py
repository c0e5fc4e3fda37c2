"""Per-kernel device time of learner steps in a normal (concurrent, graph-replayed) run via the
CUDA profiler activity API (torch.profiler / CUPTI): python tools/kprof.py [config] [steps]
Prints total / mean / share per kernel name over the profiled steps (warm caches, real overlap --
unlike an ncu launch list, which serialises and flushes caches)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from collections import defaultdict
import numpy as np, torch, synth
import paper_1911_00357_b200 as dd
from paper_1911_00357_b200.learner import Learner

cfg = sys.argv[1] if len(sys.argv) > 1 else "depth"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
hidden = int(sys.argv[3]) if len(sys.argv) > 3 else None  # e.g. 1024: the NEXT-3 LSTM on this config
ctx = dd.Context(0, 1)
c = synth.CONFIGS[cfg]
desc = dd.model_desc(c["arch"], hidden or c["hidden"]); lay = dd.param_layout(desc); P = dd.param_count(desc)
p0 = synth.init_params([(off, int(np.prod(s)), fan) for _, off, s, fan in lay], P, 0)
lrn = Learner(ctx, c["arch"], c["E"], c["T"], c["epochs"], c["minibatches"], hidden=desc.hidden, params=p0,
              normalize_adv=True)
ro = synth.rollout(c["E"], c["T"], 0, hidden=desc.hidden, obs_shape=c.get("obs"), rnn_layers=c.get("rnn_layers", 1))
pm = synth.perms(0, 0, c["epochs"], c["E"])
lrn.load_rollout(ro, pm)
for _ in range(3):
    lrn.step()
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        lrn.step()
    e1.record()
    torch.cuda.synchronize()
wall = e0.elapsed_time(e1) / steps
tot = defaultdict(float)
cnt = defaultdict(int)
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        name = ev.name.replace("(anonymous namespace)::", "")
        tot[name] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
        cnt[name] += 1
S = sum(tot.values())
print(f"{cfg}: {steps} steps, {wall:.3f} ms/step (events), kernel time sum {S / steps / 1e3:.3f} ms/step")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:40]:
    print(f"{v / steps:10.1f} us/step {100 * v / S:5.1f}% n/step {cnt[k] / steps:6.1f} mean {v / cnt[k]:8.2f} us  {k[:110]}")
