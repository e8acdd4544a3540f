"""CPU side of SURVEY §8(f) row f4: the JSON problem/solution files
(include/tsylv/io.hpp, checked by tests/cpp/test_io_dropin.cpp) and the
command-line front end's argument and file-error paths (exit code 1) — the
parts of the reference's tests/test_random_io.cpp and tests/test_cli.cpp that
need no solve.  The solving subcommands are in tests/test_gpu_cli.py."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def cli():
    from paper_1905_09539_b200 import build as b
    b.build()
    exe = b.build_cli()
    if exe is None:
        pytest.skip("nlohmann/json not found in this image")
    return exe


def run(cli, *args):
    r = subprocess.run([cli, *args], capture_output=True, text=True, timeout=120)
    return r.returncode, r.stdout + r.stderr


def test_io_files_cpp(tmp_path):
    from paper_1905_09539_b200 import build as b
    b.build()
    if b.json_include() is None:
        pytest.skip("nlohmann/json not found in this image")
    exe = str(tmp_path / "test_io_dropin")
    subprocess.run(b.cxx_user_cmd(os.path.join(ROOT, "tests", "cpp", "test_io_dropin.cpp"), exe, "-O1"), check=True)
    r = subprocess.run([exe, str(tmp_path / "io")], capture_output=True, text=True, timeout=120)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr
    assert "PASS" in r.stdout


def test_help_and_usage_errors(cli):
    rc, out = run(cli, "--help")
    assert rc == 0 and "bench-scaling" in out and "verify" in out
    rc, out = run(cli, "solve", "--help")
    assert rc == 0 and "--arithmetic" in out
    assert run(cli)[0] == 1
    assert run(cli, "frobnicate")[0] == 1
    rc, out = run(cli, "solve", "--no-such-flag")
    assert rc == 1 and "error:" in out
    assert run(cli, "solve")[0] == 1  # --in is required
    assert run(cli, "solve", "--in")[0] == 1  # value missing
    assert run(cli, "solve", "--in", "x.json", "--strategy", "fastest")[0] == 1
    assert run(cli, "solve", "--in", "x.json", "--nmin", "four")[0] == 1
    assert run(cli, "bench-scaling", "--d", "3")[0] == 1  # --n required
    assert run(cli, "bench-scaling", "--d", "3", "--n", "4,x")[0] == 1
    assert run(cli, "bench-scaling", "--d", "3", "--n", "4", "--baseline=yes")[0] == 1
    rc, out = run(cli, "bench-nmin", "--family", "laplace")
    assert rc == 1 and "--dims" in out  # neither --dims nor --d/--n


def test_bad_files_exit_1(cli, tmp_path):
    bad = tmp_path / "broken.json"
    bad.write_text("{ definitely not json")
    rc, out = run(cli, "solve", "--in", str(bad))
    assert rc == 1 and "error:" in out
    assert run(cli, "solve", "--in", str(tmp_path / "nope.json"))[0] == 1
    cplx = tmp_path / "complex.json"
    cplx.write_text(json.dumps({"family": "laplace", "complex": True, "dims": [1, 1],
                                "coeffs": [[[1]], [[[2, 0]]]], "rhs": [[1, 0]]}))
    rc, out = run(cli, "solve", "--in", str(cplx))
    assert rc == 1 and "[re, im] pair" in out
    shape = tmp_path / "shape.json"
    shape.write_text(json.dumps({"family": "laplace", "dims": [2, 2], "coeffs": [[[1]], [[1]]], "rhs": [1, 2, 3, 4]}))
    assert run(cli, "solve", "--in", str(shape))[0] == 1
