"""Complex-scalar problems (T = std::complex<double>)
on the GPU against the reference built from its own headers (oracle/_ref,
the ref_z* entry points), on inputs drawn from the reference's RandomStream:

    solve_laplace<Complex>      laplace.hpp:324-344
    solve_gsylv<Complex>        gsylv.hpp:311-331
    laplace_recursive / laplace_merged <Complex>   laplace.hpp:185-244
    gsylv_recursive / gsylv_merged <Complex>       gsylv.hpp:149-232
    solve_sylvester_tri / solve_gsylv_tri <Complex> sylvester.hpp:194-241
    mode_multiply<Complex>      tensor.hpp:187-231
    oracle::residual<Complex>   oracle.hpp:233-268

Gates: rel. difference <= 1e-10 against the reference solution and the
reference's oracle::residual of the GPU solution <= 1e-12 (north_star), plus
the reference's error and singular-witness behaviour."""
import ctypes
import os

import numpy as np
import pytest

from conftest import rel_diff

pytestmark = pytest.mark.gpu


def _crandn(shape, seed):
    g = np.random.default_rng(seed)
    return np.asfortranarray(g.standard_normal(shape) + 1j * g.standard_normal(shape))


@pytest.mark.parametrize("dims,r,mode", [((5, 7, 3), 4, 0), ((5, 7, 3), 9, 1), ((5, 7, 3), 2, 2),
                                         ((70, 65, 9), 70, 0), ((70, 65, 9), 65, 1),
                                         ((33, 130, 17), 17, 2), ((8, 3, 4, 5), 6, 3)])
def test_zmode_multiply_vs_reference(ref, gpu, dims, r, mode):
    x = _crandn(dims, 1)
    a = _crandn((r, dims[mode]), 2)
    want = ref.zmode_multiply(x, a, mode)
    got = gpu.mode_multiply(x, a, mode)
    assert got.dtype == np.complex128 and got.shape == want.shape
    assert rel_diff(got, want) <= 1e-14


@pytest.mark.parametrize("dims", [(5, 4, 3), (12, 10, 8), (33, 17, 9), (9, 8, 7, 6), (40, 40),
                                  (64, 64, 64)])
def test_zsolve_laplace_vs_reference(ref, gpu, dims):
    rs = ref.ZRandomStream(11)
    co, b = rs.laplace_problem(list(dims))
    want, info = ref.zsolve_laplace(co, b)
    rep = gpu.solve_laplace(gpu.LaplaceProblem(co, b))
    assert rep.solution.dtype == np.complex128
    assert rel_diff(rep.solution, want) <= 1e-10
    assert ref.zresidual_laplace(co, b, rep.solution) <= 1e-12
    assert rep.residual <= 1e-12 and rep.discarded_imag == 0.0
    # the device residual agrees with the reference's oracle::residual
    assert abs(rep.residual - ref.zresidual_laplace(co, b, rep.solution)) <= 1e-13


@pytest.mark.parametrize("dims", [(6, 4, 5), (20, 4, 4, 4), (40, 8, 8, 8), (17, 11), (64, 16, 16)])
def test_zsolve_gsylv_vs_reference(ref, gpu, dims):
    rs = ref.ZRandomStream(12)
    co, c, b = rs.gsylv_problem(list(dims))
    want, info = ref.zsolve_gsylv(co, c, b)
    rep = gpu.solve_gsylv(gpu.GSylvProblem(co, c, b))
    assert rel_diff(rep.solution, want) <= 1e-10
    assert ref.zresidual_gsylv(co, c, b, rep.solution) <= 1e-12
    assert abs(rep.residual - ref.zresidual_gsylv(co, c, b, rep.solution)) <= 1e-13


@pytest.mark.parametrize("dims", [(3, 4, 2), (6, 5, 4), (12, 12, 12), (5, 4, 3, 3)])
def test_zreduced_laplace_vs_reference(ref, gpu, dims):
    co, b = ref.ZRandomStream(21).reduced_laplace(list(dims))
    want_dense = ref.zdense_solve_laplace(co, b) if np.prod(dims) <= 4096 else None
    for n_min in (2, 7):
        want = ref.zlaplace_recursive(co, b, n_min)
        got = gpu.laplace_recursive(co, b, n_min)
        assert rel_diff(got, want) <= 1e-10, n_min
        if want_dense is not None:
            assert rel_diff(got, want_dense) <= 1e-9
    for n_min in (2, 26):
        want = ref.zlaplace_merged(co, b, n_min)
        got = gpu.laplace_merged(co, b, n_min)
        assert rel_diff(got, want) <= 1e-10, n_min


@pytest.mark.parametrize("dims", [(6, 4, 5), (9, 7), (8, 5, 4, 3)])
def test_zreduced_gsylv_vs_reference(ref, gpu, dims):
    co, c, b = ref.ZRandomStream(22).reduced_gsylv(list(dims))
    for n_min in (2, 6):
        want = ref.zgsylv_recursive(co, c, b, n_min)
        got = gpu.gsylv_recursive(co, c, b, n_min)
        assert rel_diff(got, want) <= 1e-10, n_min
    want = ref.zgsylv_merged(co, c, b, 13)
    got = gpu.gsylv_merged(co, c, b, 13)
    assert rel_diff(got, want) <= 1e-10


def test_zsylvester_tri_vs_reference(ref, gpu):
    rs = ref.ZRandomStream(31)
    (a1, a2), b = rs.reduced_laplace([9, 7])
    for n_min in (1, 3, 32):
        want = ref.zsolve_sylvester_tri(a1, a2, b, n_min)
        got = gpu.solve_sylvester_tri(a1, a2, b, n_min)
        assert rel_diff(got, want) <= 1e-10
    co, c, b = rs.reduced_gsylv([9, 7])
    want = ref.zsolve_gsylv_tri(co[0], c, co[1], b, 4)
    got = gpu.solve_gsylv_tri(co[0], c, co[1], b, 4)
    assert rel_diff(got, want) <= 1e-10


def test_zsolve_paths_agree(ref, gpu, monkeypatch):
    """The three reduced solves (folded eigen-decoupled, refined
    eigen-decoupled, wavefront back substitution) give the reference's X."""
    co, b = ref.ZRandomStream(41).laplace_problem([24, 20, 16])
    want, _ = ref.zsolve_laplace(co, b)
    for path in ("1", "2", "3"):
        monkeypatch.setenv("TSG_ZPATH", path)
        got = gpu.solve_laplace(gpu.LaplaceProblem(co, b)).solution
        assert rel_diff(got, want) <= 1e-10, path
    co, c, b = ref.ZRandomStream(42).gsylv_problem([24, 6, 6])
    want, _ = ref.zsolve_gsylv(co, c, b)
    for path in ("1", "2"):
        monkeypatch.setenv("TSG_ZPATH", path)
        got = gpu.solve_gsylv(gpu.GSylvProblem(co, c, b)).solution
        assert rel_diff(got, want) <= 1e-10, path


def test_zill_conditioned_reduced_takes_wavefront(ref, gpu):
    """Random triangular factors with O(1) off-diagonal entries have
    exponentially ill-conditioned eigenbases: the reduced solve must fall
    back (refined or wavefront) and still match the reference."""
    co, b = ref.ZRandomStream(51).reduced_laplace([30, 28, 26])
    want = ref.zlaplace_recursive(co, b, 7)
    got = gpu.laplace_recursive(co, b, 7)
    assert rel_diff(got, want) <= 1e-10


def _cabi_reduced(gpu, t, b, free_mode):
    from paper_1905_09539_b200._lib import TsgOpts, c_dbl_p, c_dbl_pp, lib
    from paper_1905_09539_b200.plan import Context
    ctx = Context(0)
    t = [np.asfortranarray(m, dtype=np.complex128) for m in t]
    b = np.asfortranarray(b, dtype=np.complex128)
    x = np.zeros_like(b)
    arr = (c_dbl_p * len(t))(*[m.ctypes.data_as(c_dbl_p) for m in t])
    o = TsgOpts()
    lib().tsg_default_opts(ctypes.byref(o))
    o.free_mode = free_mode
    dims = (ctypes.c_int * b.ndim)(*b.shape)
    rc = lib().tsg_zlaplace_reduced(ctx.h, b.ndim, dims, ctypes.cast(arr, c_dbl_pp),
                                    b.ctypes.data, x.ctypes.data, ctypes.byref(o), None)
    assert rc == 0, ctx.error()
    return x


def test_zfree_mode_choice_c_abi(ref, gpu):
    """Every free mode of the decoupled fibre solve (f = 0: contiguous
    fibres; f > 0: strided) through the C-ABI."""
    co, b = ref.ZRandomStream(61).laplace_problem([10, 9, 8])
    t = [ref.zschur(a)[1] for a in co]
    bt = _crandn((10, 9, 8), 5)
    want = ref.zlaplace_recursive(t, bt, 4)
    for f in (0, 1, 2):
        assert rel_diff(_cabi_reduced(gpu, t, bt, f), want) <= 1e-10, f


def test_zquasi_triangular_reduced_input(ref, gpu):
    """laplace_recursive<Complex> accepts quasi-triangular factors (2x2
    diagonal blocks) like the reference; the GPU path Schur-reduces them and
    returns the solution of the reference's dense oracle (oracle::solve).
    The reference's own complex recursion does NOT on such input (its
    complex base case mishandles 2x2 blocks: 5-11 % off the dense oracle,
    also for real-valued factors stored as complex), so the gate here is the
    dense oracle, and the reference's deviation is recorded."""
    rs = ref.RandomStream(71)
    t = [rs.quasi_triangular(n, diag_shift=3.0, pair_prob=0.7).astype(np.complex128) for n in (6, 5, 4)]
    t[1] = t[1] * (1 + 0.3j)
    b = _crandn((6, 5, 4), 6)
    dense = ref.zdense_solve_laplace(t, b)
    got = gpu.laplace_recursive(t, b, 2)
    assert rel_diff(got, dense) <= 1e-12
    assert ref.zresidual_laplace(t, b, got) <= 1e-14
    assert rel_diff(ref.zlaplace_recursive(t, b, 2), dense) > 1e-3  # the reference's deviation


def test_zerrors_and_singular(ref, gpu):
    co, b = ref.ZRandomStream(81).laplace_problem([4, 3, 2])
    p = gpu.LaplaceProblem(co, b)
    with pytest.raises(ValueError, match="real arithmetic requires real data"):
        gpu.solve_laplace(p, gpu.SolverConfig(strategy=gpu.Strategy.recursion_only,
                                              arithmetic=gpu.Arithmetic.real_quasitriangular))
    with pytest.raises(ValueError, match="merge strategy"):
        gpu.solve_laplace(p, gpu.SolverConfig(arithmetic=gpu.Arithmetic.real_quasitriangular))
    with pytest.raises(ref.RefError) as e:
        ref.zsolve_laplace(co, b, strategy=0, arithmetic=1)
    assert e.value.code == 4
    # eigenvalue sum (1+1j) + (2-1j) + (-3) = 0: singular, same witness
    ts = [np.diag([1 + 1j, 5.0]), np.diag([4.0, 2 - 1j]), np.diag([7.0, -3.0 + 0j])]
    bs = _crandn((2, 2, 2), 3)
    mn, wit, ok = ref.zcheck_solvable_laplace(ts)
    assert not ok and wit == [0, 1, 1]
    with pytest.raises(gpu.singular_error, match=r"at slots \(0,1,1\)"):
        gpu.laplace_merged(ts, bs, 8)
    with pytest.raises(gpu.singular_error):
        gpu.solve_laplace(gpu.LaplaceProblem([t.astype(np.complex128) for t in ts], bs))
    with pytest.raises(gpu.singular_error):
        gpu.laplace_recursive(ts, bs, 2)
    # non-triangular input to the merged reduced form
    with pytest.raises(gpu.dimension_error, match="must be upper triangular"):
        gpu.laplace_merged([np.ones((2, 2), complex)] * 3, bs, 8)


def test_zresidual_pinned_to_reference(ref, gpu):
    co, c, b = ref.ZRandomStream(91).gsylv_problem([12, 5, 6])
    x = _crandn((12, 5, 6), 9)
    got = gpu.residual(gpu.GSylvProblem(co, c, b), x)
    want = ref.zresidual_gsylv(co, c, b, x)
    assert abs(got - want) <= 1e-12 * want
    co, b = ref.ZRandomStream(92).laplace_problem([7, 9, 5])
    x = _crandn((7, 9, 5), 3)
    got = gpu.residual(gpu.LaplaceProblem(co, b), x)
    want = ref.zresidual_laplace(co, b, x)
    assert abs(got - want) <= 1e-12 * want
