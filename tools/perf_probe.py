"""Quick per-phase timing of the GPU path on the BASELINE configs (device-
resident inputs).  Not the bench: a development probe."""
import argparse
import time

import numpy as np
import torch

import paper_1905_09539_b200 as T
from paper_1905_09539_b200.plan import Context, Plan

CONFIGS = {
    "C1": (1, (64, 64, 64)),
    "C2": (2, (256, 256, 256)),
    "C3": (2, (24,) * 6),
    "C4": (2, (1024, 512, 256)),
    "C5": (5, (200, 40, 40, 40)),
}
PEAK = 37.07e12


def run(name, reps, tile=None, check=False):
    kind, dims = CONFIGS[name]
    t0 = time.time()
    p = T.make_problem(kind, dims, seed=1)
    t1 = time.time()
    ctx = Context()
    if kind == 5:
        q, z, s, tc = T.qz(p.coeffs[0], p.c)
        fs = [T.schur(a) for a in p.coeffs[1:]]
        plan = Plan(ctx, 1, [s] + [f[1] for f in fs], [q] + [f[0] for f in fs], Tc=tc, Z=z, tile=tile[:len(dims)] if tile else None)
    else:
        fs = [T.schur(a) for a in p.coeffs]
        plan = Plan(ctx, 0, [f[1] for f in fs], [f[0] for f in fs], tile=tile[:len(dims)] if tile else None)
    t2 = time.time()
    b = torch.from_numpy(np.ascontiguousarray(p.rhs.reshape(-1, order="F"))).cuda()
    x = torch.empty_like(b)
    reps_ = []
    for _ in range(reps):
        torch.cuda.synchronize()
        r = plan.execute_device(b.data_ptr(), x.data_ptr())
        reps_.append((r.t_fwd_ms, r.t_solve_ms, r.t_back_ms, r.t_total_ms))
    best = min(reps_, key=lambda v: v[3])
    info = plan.info()
    N = int(np.prod(dims))
    sn = sum(dims)
    f_tr = 4.0 * N * sn
    f_solve = info["flops_alg"] - f_tr
    print(f"{name} dims={dims} tiles={info['n_tiles']} tile={info['tile']} solve={plan.describe()} gen={t1-t0:.1f}s setup={t2-t1:.1f}s")
    print(f"   fwd {best[0]:.3f} ms ({f_tr/2/best[0]/1e9:.1f} TF)  solve {best[1]:.3f} ms "
          f"({f_solve/best[1]/1e9:.1f} TF alg)  back {best[2]:.3f} ms ({f_tr/2/best[2]/1e9:.1f} TF)  "
          f"total {best[3]:.3f} ms -> {info['flops_alg']/best[3]/1e9:.2f} TF = "
          f"{info['flops_alg']/best[3]/1e9/37.07*100:.1f}% of 37.07; {N/best[3]*1e3:.3e} unknowns/s")
    if check:
        xs = x.cpu().numpy().reshape(dims, order="F")
        print("   residual", T.residual(p, xs))
    plan.close()
    ctx.close()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=list(CONFIGS))
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--tile", type=str, default="")
    a = ap.parse_args()
    tiles = [None] if not a.tile else [[int(x)] * 8 for x in a.tile.split(",")]
    for c in a.configs:
        for t in tiles:
            run(c, a.reps, tile=t, check=a.check)
