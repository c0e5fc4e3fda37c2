import numpy as np, torch, synth
import paper_1911_00357_b200 as dd
from oracle import gae
ctx = dd.Context(0, 1)
for (E, T, ld) in [(2, 4, 8), (2, 4, 5), (4, 128, 132), (2, 8, 12)]:
    rng = np.random.default_rng(0)
    rew = rng.normal(size=(E, ld)).astype(np.float32)
    val = rng.normal(size=(E, ld)).astype(np.float32)
    done = np.zeros((E, ld), np.uint8)
    length = np.full(E, T, np.int32)
    r_t, v_t, d_t, l_t = [torch.from_numpy(x).cuda() for x in (rew, val, done, length)]
    adv = torch.full((E, ld), 7.0, device="cuda"); ret = torch.full((E, ld), 7.0, device="cuda")
    st = torch.zeros(3, dtype=torch.float64, device="cuda")
    dd.ddppo_gae(ctx, r_t, v_t, d_t, l_t, E, T, ld, 0.99, 0.95, adv, ret, st)
    torch.cuda.synchronize()
    a_o, r_o = gae.gae(rew, val, done, length, 0.99, 0.95)
    print(E, T, ld, "gpu", adv.cpu().numpy()[0, :min(T, 8)], "\n oracle", a_o[0, :8], "\n stats", st.cpu().numpy(), gae.adv_stats(a_o, length))
