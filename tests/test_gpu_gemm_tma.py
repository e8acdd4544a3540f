"""TMA-staged transform GEMM (csrc/gemm_tma.cu) against the cp.async kernel
and numpy on shapes with M/N/K edges, batches and the reference's
mode_multiply semantics (tensor.hpp:187-231).  The kernel choice is read once
per process (TSG_GEMM_TMA), so every setting runs in its own interpreter."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import numpy as np
import paper_1905_09539_b200 as T
rng = np.random.default_rng(5)
worst = 0.0
for dims in [(200, 66), (64, 130, 4), (66, 72, 5), (128, 64), (70, 70, 70), (256, 80, 2, 3)]:
    x = np.asfortranarray(rng.standard_normal(dims))
    for mode in range(len(dims)):
        for r in (dims[mode], 64, 90):
            a = np.asfortranarray(rng.standard_normal((r, dims[mode])))
            got = T.mode_multiply(x, a, mode)
            want = np.moveaxis(np.tensordot(a, x, axes=(1, mode)), 0, mode)
            assert got.shape == want.shape, (dims, mode, r)
            err = np.linalg.norm((got - want).ravel()) / np.linalg.norm(want.ravel())
            worst = max(worst, err)
            assert err < 1e-14, (dims, mode, r, err)
# a full pipeline through the slab chain and the programmatic launches
p = T.make_problem(2, (128, 96, 80), seed=3)
rep = T.solve_laplace(p)
res = T.residual(p, rep.solution)
assert res < 1e-12, res
print("ok", worst, res)
"""


@pytest.mark.gpu
@pytest.mark.parametrize("setting", [{"TSG_GEMM_TMA": "0"}, {"TSG_GEMM_TMA": "1"}, {"TSG_GEMM_TMA": "2"},
                                     {"TSG_GEMM_TMA": "4"}],
                         ids=["cp.async", "tma3", "tma3-early", "tma4"])
def test_tma_gemm_matches_numpy(setting):
    env = dict(os.environ, PYTHONPATH=ROOT, **setting)
    out = subprocess.run([sys.executable, "-c", SCRIPT], env=env, cwd=ROOT, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.strip().startswith("ok")
