import os
import numpy as np, torch
import oracle.ref as R
from paper_1905_09539_b200.plan import Context, Plan
ctx = Context()
for dims, tile, q in [((16, 16, 16), 16, 0.0), ((16, 16, 16), 16, 0.9), ((8, 8, 8), 8, 0.9), ((2, 2, 2), 2, 0.0)]:
    rs = R.RandomStream(5)
    T = [rs.quasi_triangular(n, 1.0, q) for n in dims]
    plan = Plan(ctx, 0, T, None, reduced_only=True, tile=[tile] * 3)
    b = torch.randn(int(np.prod(dims)), dtype=torch.float64, device="cuda"); x = torch.empty_like(b)
    ts = sorted(plan.execute_device(b.data_ptr(), x.data_ptr()).t_solve_ms for _ in range(20))
    print(os.environ.get("TSG_DBG", "0"), dims, "pairs" if q else "tri", f"med {ts[10]*1e3:.1f} us")
