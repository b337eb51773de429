"""The C++ drop-in header (include/tridpart_b200.hpp) compiles against the
reference's API shapes (CPU) and passes the reference's test expectations on
the GPU (checked against the C oracle, linked as oracle/_build/liboracle.so)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_shim.cpp")
LIBDIR = os.path.join(ROOT, "paper_2510_27351_b200", "lib")
ORCDIR = os.path.join(ROOT, "oracle", "_build")


def _build(tmp_path, oracle_mod):
    oracle_mod.port()  # ensures oracle/_build/liboracle.so exists
    exe = tmp_path / "test_shim"
    r = subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), SRC,
                        "-L", LIBDIR, "-ltridpart_b200", "-L", ORCDIR, "-loracle",
                        f"-Wl,-rpath,{LIBDIR}:{ORCDIR}", "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_shim_compiles_and_links(tmp_path, oracle_mod):
    assert _build(tmp_path, oracle_mod).exists()


@pytest.mark.gpu
def test_shim_runs_reference_expectations(tmp_path, oracle_mod):
    exe = _build(tmp_path, oracle_mod)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all passed" in r.stdout
