"""Single-tile latency probe: reduced Laplace solves small enough to be one
tile (no inter-tile updates), and 2-tile chains, timed by CUDA events."""
import numpy as np
import torch
import oracle.ref as R
from paper_1905_09539_b200.plan import Context, Plan

ctx = Context()
for dims, tile, q in [((16, 16, 16), 16, 0.0), ((16, 16, 16), 16, 0.9), ((8, 8, 8), 8, 0.0),
                      ((8, 8, 8), 8, 0.9), ((4, 4, 4), 4, 0.9), ((32, 16, 16), 16, 0.9),
                      ((32, 32, 32), 16, 0.9), ((64, 64, 64), 16, 0.9)]:
    rs = R.RandomStream(5)
    T = [rs.quasi_triangular(n, 1.0, q) for n in dims]
    plan = Plan(ctx, 0, T, None, reduced_only=True, tile=[tile] * 3)
    b = torch.randn(int(np.prod(dims)), dtype=torch.float64, device="cuda")
    x = torch.empty_like(b)
    ts = []
    for _ in range(20):
        r = plan.execute_device(b.data_ptr(), x.data_ptr())
        ts.append(r.t_solve_ms)
    print(dims, "tile", tile, "pairs" if q else "tri", plan.info()["n_tiles"], "tiles:",
          f"min {min(ts)*1e3:.1f} us  med {sorted(ts)[10]*1e3:.1f} us")
