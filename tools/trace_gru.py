"""Phase timing of the GRU forward recurrence (debug build tools/libddppo_trace.so, CTA 0 thread 0).
Slots: 0 h received, 3 MMAs issued+committed, 4 accumulator ready, 5 TMEM read, 1 after CTA barrier, 2 h sent."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1911_00357_b200._lib as L
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libddppo_trace.so"))
for name, (res, args) in L._SIGS.items():
    f = getattr(lib, name); f.restype = res; f.argtypes = args
L.lib = lib
import paper_1911_00357_b200 as dd
dd.lib = lib
import torch, synth
from paper_1911_00357_b200.learner import Learner
ctx = dd.Context(0, 1)
c = synth.CONFIGS["gps"]
desc = dd.model_desc("gps"); lay = dd.param_layout(desc); P = dd.param_count(desc)
p0 = synth.init_params([(off, int(np.prod(s)), fan) for _, off, s, fan in lay], P, 0)
lrn = Learner(ctx, "gps", c["E"], c["T"], c["epochs"], c["minibatches"], params=p0, normalize_adv=True)
lrn.load_rollout(synth.rollout(c["E"], c["T"], 0), synth.perms(0, 0, 2, c["E"]))
for _ in range(3): lrn.step()
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (8 * 128))()
lib.ddppo_debug_trace(buf, 8 * 128)
tr = np.array(buf, dtype=np.int64).reshape(128, 8)[1:-1]
med = lambda a: float(np.median(a))
print("per-step cycles (median): total %.0f | issue %.0f | mma-exec+commit %.0f | tmem-ld %.0f | "
      "->barrier %.0f | gates+send %.0f | wait-recv %.0f" % (
          med(np.diff(tr[:, 0])), med(tr[:, 3] - tr[:, 0]), med(tr[:, 4] - tr[:, 3]), med(tr[:, 5] - tr[:, 4]),
          med(tr[:, 1] - tr[:, 5]), med(tr[:, 2] - tr[:, 1]), med(tr[1:, 0] - tr[:-1, 2])))
full = (ctypes.c_longlong * (8 * 1024))()
lib.ddppo_debug_trace(full, 8 * 1024)
f = np.array(full, dtype=np.int64).reshape(1024, 8)
print("prologue cycles: tiles/X/U/TMEM-A %d | GI %d | first step starts %d after GI" % (
    f[1023, 6] - f[1023, 5], f[1023, 7] - f[1023, 6], f[0, 0] - f[1023, 7]))
print("recurrence cycles (127 steps): %d" % (f[127, 0] - f[0, 0]))
fb = (ctypes.c_longlong * (8 * 1024))()
lib.ddppo_debug_trace_bwd(fb, 8 * 1024)
b = np.array(fb, dtype=np.int64).reshape(1024, 8)
tb = b[1:126]
print("BWD per-iteration cycles (median): total %.0f | gates+sync %.0f | mma issue %.0f | mma exec %.0f | "
      "ld+send %.0f | recv wait %.0f | reduce+sync %.0f" % (
          med(np.diff(tb[:, 0])), med(tb[:, 1] - tb[:, 0]), med(tb[:, 2] - tb[:, 1]), med(tb[:, 3] - tb[:, 2]),
          med(tb[:, 4] - tb[:, 3]), med(tb[:, 5] - tb[:, 4]), med(tb[1:, 0] - tb[:-1, 5])))
print("BWD prologue %d cycles, loop %d cycles" % (b[1023, 7] - b[1023, 6], b[127, 0] - b[0, 0]))
