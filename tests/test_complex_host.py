"""Host side of the complex-scalar path, CPU only:
the drop-in's T = Complex generators draw the reference's exact instances
(random.hpp:64-223; oracle/_ref built from the reference headers), and the
complex Schur / QZ setup honours the reference's factorization contracts
(kernels.hpp:94-156)."""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def ref():
    import oracle.ref as R
    if not R.available():
        pytest.skip("oracle/_ref not built (make -C oracle)")
    return R


@pytest.fixture(scope="module")
def T():
    import paper_1905_09539_b200 as T
    return T


@pytest.mark.parametrize("dims", [[4, 3, 5], [9, 7], [6, 5, 4, 3]])
@pytest.mark.parametrize("which,fn", [("laplace", "laplace_problem"), ("reduced_laplace", "reduced_laplace"),
                                      ("gsylv", "gsylv_problem"), ("reduced_gsylv", "reduced_gsylv")])
def test_zgenerators_bit_exact(ref, T, which, fn, dims):
    p = T.random_problem(which, dims, seed=7)
    got = getattr(ref.ZRandomStream(7), fn)(dims)
    for a, w in zip(p.coeffs, got[0]):
        assert a.dtype == np.complex128 and np.array_equal(a, w)
    assert np.array_equal(p.rhs, got[-1])
    if which.endswith("gsylv"):
        assert np.array_equal(p.c, got[1])


def test_zschur_qz_contracts(ref, T):
    g = np.random.default_rng(3)
    n = 9
    a = g.standard_normal((n, n)) + 1j * g.standard_normal((n, n))
    c = g.standard_normal((n, n)) + 1j * g.standard_normal((n, n))
    u, t = T.schur(a)
    assert np.allclose(np.tril(t, -1), 0, atol=0)  # strictly triangular (zgees)
    assert np.linalg.norm(u @ t @ u.conj().T - a) <= 100 * 2.2e-16 * n * np.linalg.norm(a)
    assert np.linalg.norm(u.conj().T @ u - np.eye(n)) <= 100 * 2.2e-16 * n
    ur, tr = ref.zschur(a)
    assert np.array_equal(t, tr) and np.array_equal(u, ur)  # same LAPACK, same factors
    q, z, s, tt = T.qz(a, c)
    assert np.linalg.norm(q @ s @ z.conj().T - a) <= 100 * 2.2e-16 * n * np.linalg.norm(a)
    assert np.linalg.norm(q @ tt @ z.conj().T - c) <= 100 * 2.2e-16 * n * np.linalg.norm(c)
    assert np.array_equal(np.triu(s), s) and np.array_equal(np.triu(tt), tt)
