"""The drop-in entry points beyond solve_*/_recursive, each against the
reference function of the same name on identical inputs (oracle/_ref):

    laplace_merged       laplace.hpp:202-244
    gsylv_merged         gsylv.hpp:167-232
    solve_sylvester_tri  sylvester.hpp:194-215
    solve_gsylv_tri      sylvester.hpp:219-241
    oracle::solve / oracle::residual   oracle.hpp:205-268

including the reference's dimension_error and singular_error cases."""
import numpy as np
import pytest

from conftest import rel_diff

pytestmark = pytest.mark.gpu


def _tri(ref, seed, dims, pair_prob=0.0, shift=4.0):
    rs = ref.RandomStream(seed)
    return [rs.quasi_triangular(n, diag_shift=shift, pair_prob=pair_prob) for n in dims], rs


def _rhs(dims, seed):
    return np.asfortranarray(np.random.default_rng(seed).standard_normal(dims))


@pytest.mark.parametrize("dims", [(7, 9), (5, 6, 4), (12, 10, 8), (3, 4, 5, 3), (4, 3, 3, 2, 2)])
def test_laplace_merged_vs_reference(ref, gpu, dims):
    t, _ = _tri(ref, 5, dims)
    b = _rhs(dims, 1)
    for n_min in (2, 8, 26):
        want = ref.laplace_merged(t, b, n_min)
        got = gpu.laplace_merged(t, b, n_min)
        assert rel_diff(got, want) <= 1e-10, (n_min, rel_diff(got, want))


def test_laplace_merged_errors(ref, gpu):
    dims = (6, 5, 4)
    tq, _ = _tri(ref, 6, dims, pair_prob=0.9)   # quasi-triangular: merging needs triangular
    b = _rhs(dims, 2)
    for fn in (ref.laplace_merged, gpu.laplace_merged):
        with pytest.raises(Exception) as e:
            fn(tq, b, 8)
        assert "must be upper triangular" in str(e.value)
    t, _ = _tri(ref, 6, dims)
    with pytest.raises(gpu.dimension_error):
        gpu.laplace_merged(t, b, 0)
    with pytest.raises(ref.RefError):
        ref.laplace_merged(t, b, 0)
    with pytest.raises(gpu.dimension_error):
        gpu.laplace_merged(t, _rhs((6, 5, 3), 2), 8)
    # eigenvalue sum 1 + 3 - 4 = 0: singular on both sides
    ts = [np.diag([1.0, 2.0]), np.diag([3.0, 4.0]), np.diag([-4.0, 7.0])]
    bs = _rhs((2, 2, 2), 3)
    with pytest.raises(gpu.singular_error):
        gpu.laplace_merged(ts, bs, 8)
    with pytest.raises(ref.RefError) as e:
        ref.laplace_merged(ts, bs, 8)
    assert e.value.code == 2


@pytest.mark.parametrize("dims", [(8, 6), (6, 4, 4), (10, 5, 4, 3), (5, 3, 3, 2, 2)])
def test_gsylv_merged_vs_reference(ref, gpu, dims):
    t, rs = _tri(ref, 7, dims)
    c = rs.quasi_triangular(dims[0], diag_shift=0.3, pair_prob=0.0) * 0.25
    b = _rhs(dims, 4)
    for n_min in (2, 6, 13):
        want = ref.gsylv_merged(t, c, b, n_min)
        got = gpu.gsylv_merged(t, c, b, n_min)
        assert rel_diff(got, want) <= 1e-10, (n_min, rel_diff(got, want))


def test_gsylv_merged_errors(ref, gpu):
    dims = (6, 4, 4)
    t, rs = _tri(ref, 8, dims)
    c = np.triu(rs.quasi_triangular(6, 0.3, 0.0))
    b = _rhs(dims, 5)
    cfull = c + np.tril(np.ones((6, 6)), -1)
    for fn in (ref.gsylv_merged, gpu.gsylv_merged):
        with pytest.raises(Exception) as e:
            fn(t, cfull, b, 8)
        assert "C must be upper triangular" in str(e.value)
    tq, _ = _tri(ref, 8, dims, pair_prob=0.9)
    with pytest.raises(gpu.dimension_error):
        gpu.gsylv_merged(tq, c, b, 8)
    with pytest.raises(gpu.dimension_error):
        gpu.gsylv_merged(t, c[:5, :5], b, 8)


@pytest.mark.parametrize("r,c,pp", [(1, 1, 0.0), (9, 7, 0.5), (40, 33, 0.5), (64, 64, 0.9),
                                    (130, 20, 0.3)])
def test_solve_sylvester_tri_vs_reference(ref, gpu, r, c, pp):
    (a1, a2), _ = _tri(ref, 9 + r, (r, c), pair_prob=pp)
    b = _rhs((r, c), 6)
    for n_min in (1, 8, 32):
        want = ref.solve_sylvester_tri(a1, a2, b, n_min)
        got = gpu.solve_sylvester_tri(a1, a2, b, n_min)
        assert rel_diff(got, want) <= 1e-10, (n_min, rel_diff(got, want))


def test_solve_sylvester_tri_known_answer(gpu):
    # (3 + 2) x = 10 -> 2 (tests/test_sylvester.cpp:33-40)
    x = gpu.solve_sylvester_tri(np.array([[3.0]]), np.array([[2.0]]), np.array([[10.0]]))
    assert x[0, 0] == pytest.approx(2.0, rel=1e-15)


def test_solve_sylvester_tri_errors(ref, gpu):
    (a1, a2), _ = _tri(ref, 3, (5, 4), pair_prob=0.5)
    with pytest.raises(gpu.dimension_error):
        gpu.solve_sylvester_tri(a1, a2, _rhs((4, 5), 1))   # rhs shape
    for fn, err in ((gpu.solve_sylvester_tri, gpu.dimension_error),
                    (ref.solve_sylvester_tri, ref.RefError)):
        with pytest.raises(err):
            fn(a1, a2, _rhs((5, 4), 1), 0)        # n_min
        with pytest.raises(err):
            fn(a1 + np.tril(np.ones((5, 5)), -2), a2, _rhs((5, 4), 1))  # structure
    # lambda(A1) + conj(lambda(A2)) = 0 -> singular_error
    s1, s2 = np.diag([1.0, 2.0]), np.diag([-2.0, 5.0])
    with pytest.raises(gpu.singular_error):
        gpu.solve_sylvester_tri(s1, s2, _rhs((2, 2), 1))
    with pytest.raises(ref.RefError) as e:
        ref.solve_sylvester_tri(s1, s2, _rhs((2, 2), 1))
    assert e.value.code == 2


@pytest.mark.parametrize("r,c,pp", [(1, 1, 0.0), (9, 7, 0.5), (40, 33, 0.5), (80, 24, 0.5)])
def test_solve_gsylv_tri_vs_reference(ref, gpu, r, c, pp):
    (a1, a2), rs = _tri(ref, 20 + r, (r, c), pair_prob=pp)
    cm = np.triu(rs.quasi_triangular(r, diag_shift=0.2, pair_prob=0.0)) * 0.3
    b = _rhs((r, c), 7)
    for n_min in (1, 8, 32):
        want = ref.solve_gsylv_tri(a1, cm, a2, b, n_min)
        got = gpu.solve_gsylv_tri(a1, cm, a2, b, n_min)
        assert rel_diff(got, want) <= 1e-10, (n_min, rel_diff(got, want))


def test_solve_gsylv_tri_errors(ref, gpu):
    (a1, a2), rs = _tri(ref, 4, (5, 4), pair_prob=0.5)
    cm = np.triu(rs.quasi_triangular(5, 0.2, 0.0))
    for fn, err in ((gpu.solve_gsylv_tri, gpu.dimension_error),
                    (ref.solve_gsylv_tri, ref.RefError)):
        with pytest.raises(err):
            fn(a1, cm + np.tril(np.ones((5, 5)), -1), a2, _rhs((5, 4), 1))  # C not triangular
    with pytest.raises(gpu.dimension_error):
        gpu.solve_gsylv_tri(a1, cm, a2, _rhs((5, 5), 1))   # rhs shape
    # S + z T singular: s = 2, t = 1, tail eigenvalue -2
    with pytest.raises(gpu.singular_error):
        gpu.solve_gsylv_tri(np.array([[2.0]]), np.array([[1.0]]), np.array([[-2.0]]),
                            np.array([[1.0]]))


def test_oracle_solve_and_residual_vs_reference(ref, gpu):
    co, rhs = ref.RandomStream(31).laplace_problem([5, 4, 3])
    p = gpu.LaplaceProblem(co, rhs)
    x = gpu.oracle.solve(p)
    want = ref.dense_solve_laplace(co, rhs)
    assert rel_diff(x, want) <= 1e-12
    assert abs(gpu.oracle.residual(p, x) - ref.residual_laplace(co, rhs, x)) <= 1e-15
    co, c, rhs = ref.RandomStream(32).gsylv_problem([6, 3, 3])
    pg = gpu.GSylvProblem(co, c, rhs)
    xg = gpu.oracle.solve(pg)
    assert rel_diff(xg, ref.dense_solve_gsylv(co, c, rhs)) <= 1e-12
    # the reference's size cap (oracle.hpp:23)
    big = gpu.LaplaceProblem([np.eye(17)] * 3, np.zeros((17, 17, 17), order="F"))
    with pytest.raises(gpu.dimension_error):
        gpu.oracle.solve(big)
