"""CPU: the C-ABI library loads and exports every symbol include/tsylv_gpu.h
declares; host-only entry points (RandomStream, Schur/QZ setup, screen,
argument validation) work without a GPU."""
import os
import re

import numpy as np
import pytest

import oracle.restate as O
from conftest import ROOT, rel_diff

HDR = os.path.join(ROOT, "include", "tsylv_gpu.h")
G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def test_library_exports_every_declared_symbol():
    from paper_1905_09539_b200._lib import TSG_SYMBOLS, lib
    L = lib()
    declared = set(re.findall(r"\b(tsg_[a-z_]+)\s*\(", open(HDR).read()))
    assert declared, "no declarations parsed"
    assert declared == set(TSG_SYMBOLS)
    for name in declared:
        assert hasattr(L, name), name
    assert L.tsg_abi_version() == 1


def test_random_stream_bit_exact():
    import paper_1905_09539_b200 as T
    for seed in (1, 42, 987654321):
        rs = T.RandomStream(seed)
        assert np.array_equal(np.array([rs.uniform() for _ in range(16)]), G[f"rng{seed}_uniform"])
        assert np.array_equal(np.array([rs.normal() for _ in range(33)]), G[f"rng{seed}_normal"])


@pytest.mark.parametrize("name,kind", [("c1", 1), ("c2", 2), ("c3", 2), ("c4", 2), ("c5", 5)])
def test_make_problem_bit_exact(name, kind):
    import paper_1905_09539_b200 as T
    dims = tuple(int(v) for v in G[f"{name}_dims"])
    p = T.make_problem(kind, dims, seed=1)
    for m, a in enumerate(p.coeffs):
        assert np.array_equal(a, G[f"{name}_A{m}"])
    assert np.array_equal(p.rhs, G[f"{name}_rhs"])
    if kind == 5:
        assert np.array_equal(p.c, G[f"{name}_C"])


def test_host_schur_and_qz_contracts():
    import paper_1905_09539_b200 as T
    rs = O.RandomStream(3)
    a = O.randn_matrix(rs, 9, 9)
    c = O.randn_matrix(rs, 9, 9)
    u, t = T.schur(a)
    assert O.is_upper_quasi_triangular(t)
    assert np.abs(u @ t @ u.T - a).max() < 100 * O.U * 9 * np.abs(a).max()
    assert np.abs(u.T @ u - np.eye(9)).max() < 1e-13
    q, z, s, tt = T.qz(a, c)
    assert O.is_upper_quasi_triangular(s) and np.all(np.tril(tt, -1) == 0)
    assert np.abs(q @ s @ z.T - a).max() < 1e-12 and np.abs(q @ tt @ z.T - c).max() < 1e-12


def test_dimension_errors_are_raised_before_the_gpu():
    import paper_1905_09539_b200 as T
    with pytest.raises(T.dimension_error):
        T.solve_laplace(T.LaplaceProblem([np.eye(3)], np.zeros((3,))))
    with pytest.raises(T.dimension_error):
        T.solve_laplace(T.LaplaceProblem([np.eye(3), np.eye(4)], np.zeros((3, 5), order="F")))
    with pytest.raises(T.dimension_error):
        T.solve_gsylv(T.GSylvProblem([np.eye(3), np.eye(2)], np.eye(2), np.zeros((3, 2))))


def test_solvability_screen_host():
    import ctypes
    from paper_1905_09539_b200._lib import lib
    from paper_1905_09539_b200.api import _ptrs, _f
    t = [_f(np.diag([1.0, 2])), _f(np.diag([10.0, 20])), _f(np.diag([-21.0, 100]))]
    pp, keep = _ptrs(t)
    mn = ctypes.c_double()
    wit = (ctypes.c_int * 3)()
    ok = ctypes.c_int()
    err = ctypes.create_string_buffer(256)
    rc = lib().tsylv_check_solvable_laplace(3, (ctypes.c_int * 3)(2, 2, 2), pp, 0.0,
                                            ctypes.byref(mn), wit, ctypes.byref(ok), err, 256)
    assert rc == 0 and ok.value == 0 and list(wit) == [0, 1, 0] and mn.value == 0.0


@pytest.mark.parametrize("kind,dims", [(1, (8, 9, 10)), (2, (12, 10, 8)), (2, (5, 4, 4, 3, 3, 3)),
                                       (5, (20, 4, 4, 4))])
def test_make_problem_matches_reference_generator(ref, kind, dims):
    """The drop-in's BASELINE generator (include/tsylv/random.hpp) and the
    oracle's (the reference's own RandomStream, oracle/ref_driver.cpp
    ref_baseline_problem) give bit-identical inputs: the bench's reference
    arm builds its inputs without loading the product library."""
    import paper_1905_09539_b200 as T
    co, c, rhs = ref.baseline_problem(kind, dims, seed=3)
    p = T.make_problem(kind, dims, seed=3)
    for a, b in zip(co, p.coeffs):
        assert np.array_equal(a, b)
    assert np.array_equal(rhs, p.rhs)
    if kind == 5:
        assert np.array_equal(c, p.c)


def test_oracle_dense_solve_host(ref):
    """tsylv::oracle::solve (dense assemble + LU, host only) against the
    reference's oracle::solve on the same problem, and its size cap."""
    import paper_1905_09539_b200 as T
    co, rhs = ref.RandomStream(31).laplace_problem([5, 4, 3])
    assert rel_diff(T.oracle.solve(T.LaplaceProblem(co, rhs)), ref.dense_solve_laplace(co, rhs)) < 1e-12
    co, c, rhs = ref.RandomStream(32).gsylv_problem([6, 3, 3])
    assert rel_diff(T.oracle.solve(T.GSylvProblem(co, c, rhs)),
                    ref.dense_solve_gsylv(co, c, rhs)) < 1e-12
    with pytest.raises(T.dimension_error):
        T.oracle.solve(T.LaplaceProblem([np.eye(17)] * 3, np.zeros((17, 17, 17), order="F")))
    with pytest.raises(T.singular_error):
        T.oracle.solve(T.LaplaceProblem([np.diag([1.0, 2.0]), np.diag([-1.0, 3.0])],
                                        np.ones((2, 2), order="F")))
