"""Where does the end-to-end loop lose time against device time?  GPS config, N=1:
(a) graph-replayed steps back to back, (b) + per-step pinned H2D of the rollout arena,
(c) + per-step D2H of the statistics with the pipelined read (bench.py's e2e loop)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_1911_00357_b200 as dd
from paper_1911_00357_b200.learner import Learner

cfg = sys.argv[1] if len(sys.argv) > 1 else "gps"
K = 200
ctx = dd.Context(0, 1)
c = synth.CONFIGS[cfg]
desc = dd.model_desc(c["arch"]); lay = dd.param_layout(desc); P = dd.param_count(desc)
p0 = synth.init_params([(off, int(np.prod(s)), fan) for _, off, s, fan in lay], P, 0)
lrn = Learner(ctx, c["arch"], c["E"], c["T"], c["epochs"], c["minibatches"], params=p0, normalize_adv=True)
ro = synth.rollout(c["E"], c["T"], 0, hidden=desc.hidden, obs_shape=c.get("obs"), rnn_layers=c.get("rnn_layers", 1))
pm = synth.perms(0, 0, c["epochs"], c["E"])
hb = lrn.pinned_host_buffers()
for k in hb:
    if k not in ("__arena__", "perms"):
        hb[k].copy_(torch.from_numpy(np.ascontiguousarray(ro[k])).reshape(hb[k].shape))
lrn.load_rollout(hb, pm)
stream = torch.cuda.current_stream()
for _ in range(5):
    lrn.step(stream)
torch.cuda.synchronize()


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record(stream)
    fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K, (time.perf_counter() - t0) * 1e3 / K


def a():
    for _ in range(K):
        lrn.step(stream)


def b():
    for _ in range(K):
        lrn.load_rollout(hb, pm, non_blocking=True)
        lrn.step(stream)


stats_dev = [torch.zeros_like(lrn.stats) for _ in range(2)]
stats_host = [torch.zeros(lrn.stats.shape, dtype=lrn.stats.dtype).pin_memory() for _ in range(2)]
copy_stream = torch.cuda.Stream()
done = [torch.cuda.Event() for _ in range(2)]


def cfn():
    for i in range(K):
        lrn.load_rollout(hb, pm, non_blocking=True)
        lrn.step(stream, stats=stats_dev[i % 2])
        copy_stream.wait_stream(stream)
        with torch.cuda.stream(copy_stream):
            stats_host[i % 2].copy_(stats_dev[i % 2], non_blocking=True)
            done[i % 2].record(copy_stream)
        if i > 0:
            done[(i - 1) % 2].synchronize()
    done[(K - 1) % 2].synchronize()


def d_alt_stats():  # alternating stats buffers, no D2H
    for i in range(K):
        lrn.load_rollout(hb, pm, non_blocking=True)
        lrn.step(stream, stats=stats_dev[i % 2])


def e_d2h_no_wait():  # D2H on the copy stream, no host wait
    for i in range(K):
        lrn.load_rollout(hb, pm, non_blocking=True)
        lrn.step(stream, stats=stats_dev[i % 2])
        copy_stream.wait_stream(stream)
        with torch.cuda.stream(copy_stream):
            stats_host[i % 2].copy_(stats_dev[i % 2], non_blocking=True)


def f_d2h_same_stream():  # D2H on the launching stream, host waits one step behind
    ev = [torch.cuda.Event() for _ in range(2)]
    for i in range(K):
        lrn.load_rollout(hb, pm, non_blocking=True)
        lrn.step(stream, stats=stats_dev[i % 2])
        stats_host[i % 2].copy_(stats_dev[i % 2], non_blocking=True)
        ev[i % 2].record(stream)
        if i > 0:
            ev[(i - 1) % 2].synchronize()
    ev[(K - 1) % 2].synchronize()


def host_only():
    for _ in range(K):
        lrn.load_rollout(hb, pm, non_blocking=True)


for name, fn in [("a steps only", a), ("b + H2D", b), ("c + H2D + D2H pipelined", cfn),
                 ("c again (graphs cached)", cfn), ("d alternating stats", d_alt_stats),
                 ("e D2H no host wait", e_d2h_no_wait), ("f D2H same stream", f_d2h_same_stream),
                 ("a steps only", a)]:
    dev, wall = timed(fn)
    print(f"{name:28s} device {dev:.4f} ms/step  host wall {wall:.4f} ms/step", flush=True)
t0 = time.perf_counter()
for _ in range(K):
    lrn.step(stream)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"host enqueue cost of step(): {(t1 - t0) * 1e3 / K:.4f} ms/step (may block when the queue fills)")
