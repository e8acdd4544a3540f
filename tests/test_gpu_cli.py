"""GPU side of SURVEY §8(f) row f4: the command-line front end
(tools/tsylv_cli.cpp -> paper_1905_09539_b200/bin/tsylv) driven the way the
reference's tests/test_cli.cpp drives its own: solve from a problem file to a
solution file (checked against the closed form and the dense oracle), the
strategy/cutoff flags, singular operators exit 2, the bench CSVs and the
verify suite with its timing-free solution files."""
import json
import subprocess

import numpy as np
import pytest

from conftest import rel_diff
from oracle import restate as R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cli(gpu):
    from paper_1905_09539_b200 import build as b
    exe = b.build_cli()
    if exe is None:
        pytest.skip("nlohmann/json not found in this image")
    return exe


def run(cli, *args, timeout=600):
    r = subprocess.run([cli, *map(str, args)], capture_output=True, text=True, timeout=timeout)
    return r.returncode, r.stdout, r.stderr


def write_problem(path, coeffs, rhs, c=None):
    doc = {"family": "gsylv" if c is not None else "laplace", "complex": False, "dims": list(rhs.shape),
           "coeffs": [a.tolist() for a in coeffs], "rhs": rhs.reshape(-1, order="F").tolist()}
    if c is not None:
        doc["c_coeff"] = c.tolist()
    path.write_text(json.dumps(doc))
    return path


def read_solution(path):
    doc = json.loads(path.read_text())
    return np.array(doc["solution"]).reshape(doc["dims"], order="F"), doc


def test_solve_diagonal_closed_form(cli, tmp_path):
    a0, a1 = np.diag([1.0, 2.0]), np.diag([10.0, 11.0, 12.0])
    b = np.array([[1.0 + i + 2 * j for j in range(3)] for i in range(2)])
    inp = write_problem(tmp_path / "diag.json", [a0, a1], b)
    out = tmp_path / "diag_sol.json"
    rc, so, se = run(cli, "solve", "--in", inp, "--out", out)
    assert rc == 0, se
    for line in ("family: laplace", "dims: 2x3", "residual:", "reduction_s:", "recursion_s:", "back_transform_s:"):
        assert line in so
    x, doc = read_solution(out)
    want = b / (np.diag(a0)[:, None] + np.diag(a1)[None, :])
    assert rel_diff(x, want) <= 1e-14
    assert doc["report"]["strategy"] == "merge" and "timings" in doc["report"]
    assert doc["report"]["residual"] <= 1e-14


@pytest.mark.parametrize("family", ["laplace", "gsylv"])
def test_solve_random_vs_dense_oracle(cli, tmp_path, family):
    rs = R.RandomStream(71)
    dims = [5, 4, 3]
    coeffs = [R.randn_matrix(rs, n, n) + 2 * n * np.eye(n) for n in dims]
    rhs = R.randn_tensor(rs, dims)
    c = R.randn_matrix(rs, 5, 5) + 10 * np.eye(5) if family == "gsylv" else None
    inp = write_problem(tmp_path / f"{family}.json", coeffs, rhs, c)
    out = tmp_path / f"{family}_sol.json"
    rc, so, se = run(cli, "solve", "--in", inp, "--out", out, "--strategy", "recursion", "--nmin", 2, "--arithmetic",
                     "real")
    assert rc == 0, se
    assert f"family: {family}" in so and "strategy: recursion" in so and "n_min: 2" in so
    assert "discarded_imag: 0.000000e+00" in so
    x, doc = read_solution(out)
    ref = R.dense_solve_laplace(coeffs, rhs) if c is None else R.dense_solve_gsylv(coeffs, c, rhs)
    assert rel_diff(x, ref) <= 1e-12
    res = R.residual_laplace(coeffs, rhs, x) if c is None else R.residual_gsylv(coeffs, c, rhs, x)
    assert res <= 1e-14 and abs(doc["report"]["residual"] - res) <= 1e-15 + 0.5 * res
    # merge with complex arithmetic: the same unique solution
    rc, so, se = run(cli, "solve", "--in", inp, "--out", tmp_path / "m.json")
    assert rc == 0, se
    assert rel_diff(read_solution(tmp_path / "m.json")[0], ref) <= 1e-12
    # merge cannot run in real quasi-triangular arithmetic: bad input
    assert run(cli, "solve", "--in", inp, "--arithmetic", "real")[0] == 1


def test_singular_exit_2(cli, tmp_path):
    a0, a1 = np.diag([1.0, 2.0]), np.diag([-1.0, 5.0])  # 1 + (-1) = 0
    b = np.zeros((2, 2))
    b[0, 0] = 1
    rc, so, se = run(cli, "solve", "--in", write_problem(tmp_path / "sing.json", [a0, a1], b))
    assert rc == 2 and "singular" in se
    # gsylv: I (x) A_0 + A_1 (x) C with C = I has eigenvalue 1 + (-1) * 1 = 0
    rc, so, se = run(cli, "solve", "--in", write_problem(tmp_path / "gsing.json", [a0, a1], b, c=np.eye(2)))
    assert rc == 2 and "singular" in se


def test_bench_nmin_csv(cli, tmp_path):
    csv = tmp_path / "nmin.csv"
    rc, so, se = run(cli, "bench-nmin", "--family", "laplace", "--d", 3, "--n", 6, "--nmin", "2,4", "--strategy", "both",
                     "--seed", 5, "--reps", 1, "--out", csv)
    assert rc == 0, se
    text = csv.read_bytes().decode()
    assert text == so
    assert text.startswith("family,d,n,n_min,strategy,wall_mean_s,wall_min_s,residual,discarded_imag,status,seed\n")
    assert text.count("\n") == 5 and "\r" not in text
    assert "laplace,3,6,2,recursion," in text and "laplace,3,6,4,merge," in text and ",ok,5" in text
    rc, so, se = run(cli, "bench-nmin", "--family", "gsylv", "--dims", "7,5,4", "--strategy", "merge", "--reps", 1)
    assert rc == 0, se
    assert so.count("\n") == 2 and "gsylv,3,7," in so


def test_bench_scaling_with_baseline_and_oom(cli):
    rc, so, se = run(cli, "bench-scaling", "--family", "gsylv", "--d", 4, "--n", "3,4", "--baseline", "--seed", 9,
                     "--reps", 1, "--mem-cap-bytes", 40000)
    assert rc == 0, se
    assert "gsylv,4,3,0,sylvester" in so  # 27^2 doubles x3 fits 40 KB
    assert ",oom,9" in so  # 64^2 doubles x3 does not


def _zarr(v):
    a = np.asarray(v, dtype=float)
    return a[..., 0] + 1j * a[..., 1]


def test_verify_writes_timing_free_files(cli, ref, tmp_path):
    """run_verify (bench.hpp:255-352): the reference's complex reduced-form
    suite; the files must hold the reference's own instances (bit-identical
    envelopes) and solutions within 1e-10 of the reference's run_verify."""
    out = tmp_path / "verify_out"
    rc, so, se = run(cli, "verify", "--seed", 12, "--count", 2, "--out", out)
    assert rc == 0, se + so
    assert "instances: 4" in so and "verify: PASS" in so
    ref_out = tmp_path / "verify_ref"
    ref_out.mkdir()
    vr = ref.run_verify(12, 2, str(ref_out))
    assert vr["pass"] and vr["instances"] == 4
    for name in ("verify_laplace_0.json", "verify_laplace_1.json", "verify_gsylv_0.json", "verify_gsylv_1.json"):
        assert (out / name).exists()
        mine, theirs = json.loads((out / name).read_text()), json.loads((ref_out / name).read_text())
        assert mine["complex"] is True
        for key in ("family", "complex", "dims", "coeffs", "rhs") + (("c_coeff",) if "gsylv" in name else ()):
            assert mine[key] == theirs[key], (name, key)
        assert rel_diff(_zarr(mine["solution"]), _zarr(theirs["solution"])) <= 1e-10, name
        assert mine["report"]["n_min"] == theirs["report"]["n_min"]
        assert mine["report"]["strategy"] == theirs["report"]["strategy"] == "merge"
    text = (out / "verify_laplace_0.json").read_text()
    assert "timings" not in text
    doc = json.loads((out / "verify_gsylv_1.json").read_text())
    co = [_zarr(a) for a in doc["coeffs"]]
    rhs = _zarr(doc["rhs"]).reshape(doc["dims"], order="F")
    x = _zarr(doc["solution"]).reshape(doc["dims"], order="F")
    assert ref.zresidual_gsylv(co, _zarr(doc["c_coeff"]), rhs, x) <= 1e-12
    # an impossible tolerance fails the suite with exit code 4
    rc, so, se = run(cli, "verify", "--seed", 12, "--count", 1, "--tol", 1e-300)
    assert rc == 4 and "verify: FAIL" in so


def test_solve_complex_problem_file(cli, ref, tmp_path):
    """A complex problem file ("complex": true, [re, im] scalars) solves on
    the GPU to the reference's solve_laplace<Complex> / solve_gsylv<Complex>."""
    rs = ref.ZRandomStream(17)
    for family in ("laplace", "gsylv"):
        if family == "laplace":
            co, b = rs.laplace_problem([6, 5, 4])
            c = None
            want, _ = ref.zsolve_laplace(co, b)
        else:
            co, c, b = rs.gsylv_problem([6, 5, 4])
            want, _ = ref.zsolve_gsylv(co, c, b)
        pair = lambda a: np.stack([a.real, a.imag], axis=-1).tolist()  # noqa: E731
        doc = {"family": family, "complex": True, "dims": list(b.shape), "coeffs": [pair(a) for a in co],
               "rhs": pair(b.reshape(-1, order="F"))}
        if c is not None:
            doc["c_coeff"] = pair(c)
        inp = tmp_path / f"z{family}.json"
        inp.write_text(json.dumps(doc))
        out = tmp_path / f"z{family}_sol.json"
        rc, so, se = run(cli, "solve", "--in", inp, "--out", out)
        assert rc == 0, se + so
        sol = json.loads(out.read_text())
        assert sol["complex"] is True
        x = _zarr(sol["solution"]).reshape(sol["dims"], order="F")
        assert rel_diff(x, want) <= 1e-10
        assert sol["report"]["residual"] <= 1e-12
