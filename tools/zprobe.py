"""One complex solve (Z2 = Laplace 256^3 or Z5 = gsylv 200x40^3, bench.COMPLEX_CONFIGS) for ncu captures."""
import sys

import paper_1905_09539_b200 as T

fam, dims = {"Z2": ("laplace", (256, 256, 256)), "Z5": ("gsylv", (200, 40, 40, 40))}[sys.argv[1] if len(sys.argv) > 1 else "Z2"]
p = T.random_problem(fam, dims, seed=1)
solve = T.solve_laplace if fam == "laplace" else T.solve_gsylv
for _ in range(2):
    rep = solve(p)
g = rep.gpu
print(fam, dims, {k: round(g[k], 3) for k in ("fwd_ms", "solve_ms", "back_ms")}, "residual", rep.residual)
