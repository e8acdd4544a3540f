"""The GPU solvability screen (tsg_screen_laplace / tsg_screen_gsylv,
csrc/screen.cu) against the reference's own
check_solvable_laplace / check_solvable_gsylv (laplace.hpp:28-43,
gsylv.hpp:31-50, solvability.hpp:31-116) on identical reduced factors:
minimum magnitude (to a few ulps of |.|), witness (the first minimum in the
reference's scan order), solvable flag; exact ties and singular operators;
the BASELINE configurations C1, C2, C5 at full size, and C3/C4 (191M / 134M
tuples) against the drop-in's threaded host scan."""
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _laplace_factors(gpu, kind, dims, seed):
    p = gpu.make_problem(kind, dims, seed=seed)
    return [gpu.schur(a)[1] for a in p.coeffs]


def _gsylv_factors(gpu, dims, seed):
    p = gpu.make_problem(5, dims, seed=seed)
    q, z, s, tc = gpu.qz(p.coeffs[0], p.c)
    return s, tc, [gpu.schur(a)[1] for a in p.coeffs[1:]]


@pytest.mark.parametrize("kind,dims", [(1, (64, 64, 64)), (2, (256, 256, 256)), (2, (12, 10, 8)),
                                       (2, (7, 6, 5, 4, 3)), (1, (9, 48))])
def test_screen_laplace_vs_reference(ref, gpu, kind, dims):
    t = _laplace_factors(gpu, kind, dims, 1)
    t0 = time.perf_counter()
    mn, wit, ok = gpu.screen_laplace(t)
    t1 = time.perf_counter()
    rmn, rwit, rok = ref.check_solvable_laplace(t)
    t2 = time.perf_counter()
    print(f"{dims}: gpu {mn:.17g} {wit} ({(t1 - t0) * 1e3:.1f} ms)  reference {rmn:.17g} {rwit} "
          f"({(t2 - t1) * 1e3:.0f} ms)")
    assert ok and rok
    assert abs(mn - rmn) <= 4e-16 * rmn
    assert wit == rwit


@pytest.mark.parametrize("dims", [(200, 40, 40, 40), (20, 4, 4, 4), (33, 7, 7), (16, 3, 3, 3, 3)])
def test_screen_gsylv_vs_reference(ref, gpu, dims):
    s, tc, tails = _gsylv_factors(gpu, dims, 1)
    t0 = time.perf_counter()
    mn, wit, ok = gpu.screen_gsylv(s, tc, tails)
    t1 = time.perf_counter()
    rmn, rwit, rok = ref.check_solvable_gsylv([s] + tails, tc)
    t2 = time.perf_counter()
    print(f"{dims}: gpu {mn:.17g} {wit} ({(t1 - t0) * 1e3:.1f} ms)  reference {rmn:.17g} {rwit} "
          f"({(t2 - t1) * 1e3:.0f} ms)")
    assert ok and rok
    assert abs(mn - rmn) <= 1e-14 * max(rmn, 1e-300)
    assert wit == rwit


def test_screen_ties_and_singular(ref, gpu):
    """Exact zeros and ties: the witness is the FIRST tuple in odometer order."""
    t = [np.diag([1.0, 2.0]), np.diag([10.0, 20.0]), np.diag([-21.0, 100.0])]
    assert gpu.screen_laplace(t) == (0.0, [0, 1, 0], False)
    # every tuple of equal magnitude: the first (all zeros) wins
    t = [np.diag([1.0, 1.0, 1.0]), np.diag([2.0, 2.0]), np.diag([3.0, 3.0, 3.0, 3.0])]
    mn, wit, ok = gpu.screen_laplace(t)
    assert (mn, wit) == (6.0, [0, 0, 0]) and ok
    assert ref.check_solvable_laplace(t)[:2] == (6.0, [0, 0, 0])
    # gsylv: S + z Tc singular for z = 1 * (-2) on block 1
    s = np.array([[1.0, 5.0], [0.0, 4.0]])
    tc = np.array([[1.0, 0.0], [0.0, 2.0]])
    tails = [np.diag([3.0, 1.0]), np.diag([-2.0, 7.0])]
    mn, wit, ok = gpu.screen_gsylv(s, tc, tails)
    rmn, rwit, rok = ref.check_solvable_gsylv([s] + tails, tc)
    assert (mn, wit, ok) == (rmn, rwit, rok) == (0.0, [1, 1, 0], False)


@pytest.mark.parametrize("kind,dims", [(2, (24,) * 6), (2, (1024, 512, 256))])
def test_screen_large_vs_host(gpu, kind, dims):
    """C3 / C4: against the drop-in's threaded host scan (the reference's
    sequential loop takes minutes here)."""
    import ctypes
    from paper_1905_09539_b200._lib import lib
    from paper_1905_09539_b200.api import _ptrs, _f
    t = [_f(m) for m in _laplace_factors(gpu, kind, dims, 1)]
    t0 = time.perf_counter()
    mn, wit, ok = gpu.screen_laplace(t)
    t1 = time.perf_counter()
    pp, keep = _ptrs(t)
    hm, hok = ctypes.c_double(), ctypes.c_int()
    hw = (ctypes.c_int * len(t))()
    err = ctypes.create_string_buffer(256)
    rc = lib().tsylv_check_solvable_laplace(len(t), (ctypes.c_int * len(t))(*dims), pp, 0.0, ctypes.byref(hm),
                                            hw, ctypes.byref(hok), err, 256)
    t2 = time.perf_counter()
    assert rc == 0
    print(f"{dims}: gpu {mn:.17g} {wit} ({(t1 - t0) * 1e3:.1f} ms)  host {hm.value:.17g} {list(hw)} "
          f"({(t2 - t1) * 1e3:.0f} ms)")
    assert ok and hok.value
    assert abs(mn - hm.value) <= 4e-16 * hm.value
    assert wit == list(hw)
