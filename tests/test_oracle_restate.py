"""CPU: pin the numpy restatement oracle (oracle/restate.py) against the
golden fixtures generated from the reference itself, and (when built)
against the reference library directly."""
import os

import numpy as np
import pytest

import oracle.restate as O
from conftest import rel_diff

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def coeffs(prefix, d):
    return [G[f"{prefix}_A{m}"] for m in range(d)]


def test_random_stream_known_answers():
    for seed in (1, 42, 987654321):
        rs = O.RandomStream(seed)
        assert np.array_equal(np.array([rs.uniform() for _ in range(16)]), G[f"rng{seed}_uniform"])
        assert np.array_equal(np.array([rs.normal() for _ in range(33)]), G[f"rng{seed}_normal"])


@pytest.mark.parametrize("name,kind", [("c1", 1), ("c2", 2), ("c3", 2), ("c4", 2), ("c5", 5)])
def test_baseline_generators_bit_exact(name, kind):
    dims = tuple(int(v) for v in G[f"{name}_dims"])
    co, c, rhs = O.baseline_problem(kind, dims, 1)
    for m, a in enumerate(co):
        assert np.array_equal(a, G[f"{name}_A{m}"])
    assert np.array_equal(rhs, G[f"{name}_rhs"])
    if kind == 5:
        assert np.array_equal(c, G[f"{name}_C"])


@pytest.mark.parametrize("i,d", [(0, 2), (1, 3), (2, 4), (3, 5)])
def test_laplace_recursive_matches_reference(i, d):
    t = coeffs(f"lr{i}", d)
    got = O.laplace_recursive(t, G[f"lr{i}_B"], 2)
    assert rel_diff(got, G[f"lr{i}_X"]) < 1e-12


def test_laplace_recursive_quasi_matches_reference():
    got = O.laplace_recursive(coeffs("lq", 3), G["lq_B"], 3)
    assert rel_diff(got, G["lq_X"]) < 1e-12


@pytest.mark.parametrize("i,d", [(0, 2), (1, 3), (2, 4)])
def test_gsylv_recursive_matches_reference(i, d):
    got = O.gsylv_recursive(coeffs(f"gr{i}", d), G[f"gr{i}_C"], G[f"gr{i}_B"], 2)
    assert rel_diff(got, G[f"gr{i}_X"]) < 1e-12


def test_mode_multiply_matches_reference():
    for m in range(3):
        assert rel_diff(O.mode_multiply(G["mm_X"], G[f"mm_A{m}"], m), G[f"mm_Y{m}"]) < 1e-14


@pytest.mark.parametrize("name,kind", [("c1", 1), ("c2", 2), ("c4", 2), ("c5", 5)])
def test_pipeline_matches_reference(name, kind):
    dims = tuple(int(v) for v in G[f"{name}_dims"])
    co = coeffs(name, len(dims))
    rhs = G[f"{name}_rhs"]
    if kind == 5:
        x = O.solve_gsylv(co, G[f"{name}_C"], rhs)
        assert O.residual_gsylv(co, G[f"{name}_C"], rhs, x) < 1e-13
    else:
        x = O.solve_laplace(co, rhs)
        assert O.residual_laplace(co, rhs, x) < 1e-13
    # both reference arithmetics agree with the restatement
    assert rel_diff(x, G[f"{name}_X_default"]) < 1e-10
    assert rel_diff(x, G[f"{name}_X_real"]) < 1e-10


def test_dense_oracle_and_residual():
    co = coeffs("c2", 3)
    rhs = G["c2_rhs"]
    x = O.dense_solve_laplace(co, rhs)
    assert rel_diff(x, G["c2_X_default"]) < 1e-12
    assert O.residual_laplace(co, rhs, x) < 1e-14
    assert abs(O.residual_laplace(co, rhs, G["c2_X_real"]) - G["c2_residual"][1]) < 1e-15


def test_closed_forms():
    # diagonal Laplace: X = B / (d0_i + d1_j + d2_k)   (test_laplace.cpp:218-231)
    d0, d1, d2 = [1.0, 2, 3], [4.0, 5], [6.0, 7, 8, 9]
    rhs = O.randn_tensor(O.RandomStream(1008), (3, 2, 4))
    x = O.solve_laplace([np.diag(d0), np.diag(d1), np.diag(d2)], rhs)
    want = rhs / (np.array(d0)[:, None, None] + np.array(d1)[None, :, None] + np.array(d2)[None, None, :])
    assert np.allclose(x, want, rtol=1e-12, atol=0)
    # 1x1 Sylvester: (3 + 2) x = 10 -> 2   (test_sylvester.cpp:33-40)
    assert O.laplace_recursive([np.array([[3.0]]), np.array([[2.0]])], np.array([[10.0]]), 1)[0, 0] == 2.0


def test_singular_screen_witness():
    # laplace spectra {1,5}, {-1,7}: 1 + (-1) = 0 at slots (0,0)  (test_laplace.cpp:37-47)
    m, w = O.min_kron_sum([[1, 5], [-1, 7]])
    assert m == 0.0 and w == [0, 0]
    m, w = O.min_kron_sum([[1, 2], [10, 20], [-21, 100]])
    assert w == [0, 1, 0]


def test_against_reference_library(ref):
    rs = ref.RandomStream(77)
    t, b = rs.reduced_laplace([5, 4, 6])
    assert rel_diff(O.laplace_recursive(t, b, 2), ref.laplace_recursive(t, b, 2)) < 1e-12
    u, tt = ref.schur(t[0] + np.tril(rs.randn(25).reshape(5, 5), -1))
    assert O.is_upper_quasi_triangular(tt)
