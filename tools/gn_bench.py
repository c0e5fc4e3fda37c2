"""GroupNorm kernel timing at the Depth / RGB-D layer shapes (F = 256 frames, channels-last).
Usage: python tools/gn_bench.py [label]  -> one line per shape: fwd us, fwd+bwd us (CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1911_00357_b200 as dd

SHAPES = [(4096, 32), (1024, 32), (1024, 128), (256, 64), (256, 256), (64, 128), (64, 512), (16, 256),
          (16, 1024), (256, 32), (64, 64), (16, 128), (4, 256)]


def main():
    label = sys.argv[1] if len(sys.argv) > 1 else ""
    ctx = dd.Context(0, 1)
    F = 256
    for HW, C in SHAPES:
        y = torch.randn(F, HW, C, device="cuda")
        r = torch.randn(F, HW, C, device="cuda")
        g = torch.rand(C, device="cuda") + 0.5
        b = torch.randn(C, device="cuda")
        z = torch.empty_like(y)
        dy = torch.empty_like(y)
        dz = torch.randn_like(y)
        st = torch.empty(F, 16, 2, device="cuda")
        dg = torch.empty(C, device="cuda")
        db = torch.empty(C, device="cuda")
        res = []
        for bwd in (False, True):
            keep = []
            for _ in range(3):
                keep.append(dd.ddppo_debug_groupnorm(ctx, y, g, b, F, HW, C, True, z, st, residual=r,
                                                     dz=dz if bwd else None, dy=dy if bwd else None,
                                                     dgamma=dg if bwd else None, dbeta=db if bwd else None))
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n = 20
            e0.record()
            for _ in range(n):
                keep.append(dd.ddppo_debug_groupnorm(ctx, y, g, b, F, HW, C, True, z, st, residual=r,
                                                     dz=dz if bwd else None, dy=dy if bwd else None,
                                                     dgamma=dg if bwd else None, dbeta=db if bwd else None))
            e1.record()
            torch.cuda.synchronize()
            res.append(e0.elapsed_time(e1) * 1e3 / n)
        mb = F * HW * C * 4 / 1e6
        print(f"{label} HW={HW:5d} C={C:5d} {mb:7.1f}MB fwd {res[0]:8.1f} us  fwd+bwd {res[1]:8.1f} us", flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
