"""Idle time between consecutive kernels of the learner step's critical stream (graph replay, CUPTI
timestamps via torch.profiler's Chrome trace): python tools/gaps.py [config] [steps]
Prints, per stream, kernels per step, busy time, the summed gaps between a kernel's end and the next
kernel's start, and the gap distribution -- the launch / ramp overhead that programmatic dependent
launch or kernel fusion could recover."""
import json, os, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from collections import defaultdict
import numpy as np, torch, synth
import paper_1911_00357_b200 as dd
from paper_1911_00357_b200.learner import Learner

cfg = sys.argv[1] if len(sys.argv) > 1 else "depth"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ctx = dd.Context(0, 1)
c = synth.CONFIGS[cfg]
desc = dd.model_desc(c["arch"], c["hidden"]); lay = dd.param_layout(desc); P = dd.param_count(desc)
p0 = synth.init_params([(off, int(np.prod(s)), fan) for _, off, s, fan in lay], P, 0)
lrn = Learner(ctx, c["arch"], c["E"], c["T"], c["epochs"], c["minibatches"], hidden=desc.hidden, params=p0,
              normalize_adv=True)
ro = synth.rollout(c["E"], c["T"], 0, hidden=desc.hidden, obs_shape=c.get("obs"), rnn_layers=c.get("rnn_layers", 1))
lrn.load_rollout(ro, synth.perms(0, 0, c["epochs"], c["E"]))
for _ in range(3):
    lrn.step()
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(steps):
        lrn.step()
    torch.cuda.synchronize()
path = os.path.join(tempfile.mkdtemp(), "trace.json")
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
by_stream = defaultdict(list)
for e in ev:
    by_stream[e["args"].get("stream", e.get("tid"))].append((e["ts"], e["ts"] + e["dur"], e["name"]))
t0 = min(e["ts"] for e in ev)
t1 = max(e["ts"] + e["dur"] for e in ev)
print(f"{cfg}: {steps} steps, span {(t1 - t0) / steps / 1e3:.3f} ms/step")
for s, ks in sorted(by_stream.items(), key=lambda kv: -len(kv[1])):
    ks.sort()
    busy = sum(b - a for a, b, _ in ks)
    gaps = np.array([max(0.0, ks[i + 1][0] - ks[i][1]) for i in range(len(ks) - 1)])
    small = gaps[gaps < 20.0]  # back-to-back dependent launches (larger gaps: waiting on another stream)
    print(f"stream {s}: {len(ks) / steps:.0f} kernels/step, busy {busy / steps / 1e3:.3f} ms/step, "
          f"gaps {gaps.sum() / steps / 1e3:.3f} ms/step (< 20 us: {small.sum() / steps / 1e3:.3f} ms/step, "
          f"median {np.median(small) if len(small) else 0:.2f} us, p90 {np.percentile(small, 90) if len(small) else 0:.2f} us)")

main = max(by_stream.items(), key=lambda kv: sum(b - a for a, b, _ in kv[1]))[1]
tot = defaultdict(float)
cnt = defaultdict(int)
for a, b, n in main:
    n = n.replace("(anonymous namespace)::", "").split("(")[0][:70]
    tot[n] += b - a
    cnt[n] += 1
print("busiest stream, top kernels (us/step, launches/step):")
for n, v in sorted(tot.items(), key=lambda kv: -kv[1])[:15]:
    print(f"  {v / steps:8.1f} {cnt[n] / steps:6.1f}  {n}")
