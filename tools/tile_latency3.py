import os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import oracle.ref as R
from paper_1905_09539_b200.plan import Context, Plan
ctx = Context()
for dims, tile, q in [((8, 8, 8), 8, 0.0), ((8, 8, 8), 8, 0.9), ((16, 8, 8), 8, 0.9), ((16, 16, 16), 8, 0.9), ((2, 2, 2), 8, 0.0)]:
    rs = R.RandomStream(5)
    T = [rs.quasi_triangular(n, 1.0, q) for n in dims]
    plan = Plan(ctx, 0, T, None, reduced_only=True, tile=[tile] * 3)
    b = torch.randn(int(np.prod(dims)), dtype=torch.float64, device="cuda"); x = torch.empty_like(b)
    ts = sorted(plan.execute_device(b.data_ptr(), x.data_ptr()).t_solve_ms for _ in range(30))
    print(os.environ.get("TSG_PROF", ""), dims, "pairs" if q else "tri", plan.info()["n_tiles"], f"med {ts[15]*1e3:.1f} us")
