"""The glibc-faithful exp/log/sincos ports (csrc/mcg_libm.h) agree bit for bit
with the live glibc libm on millions of random arguments per range (host
build; the GPU tests repeat the comparison for the device build)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def checker(tmp_path_factory):
    out = tmp_path_factory.mktemp("lpc") / "libm_port_check"
    subprocess.run(["gcc", "-O2", "-mfma", "-ffp-contract=off",
                    "-I", os.path.join(ROOT, "paper_2411_16445_b200", "csrc"),
                    os.path.join(ROOT, "tests", "native", "libm_port_check.c"),
                    "-o", str(out), "-lm"], check=True)
    return str(out)


@pytest.mark.parametrize("seed", [1, 2])
def test_port_matches_glibc(checker, seed):
    r = subprocess.run([checker, "1000000", str(seed)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:] + r.stdout
    assert "0 mismatches" in r.stdout


def test_runtime_libm_pin():
    """libmcg's load-time pin: this host's libm build-id, its FMA ifunc
    variant and a differential run all agree with the device ports' tables."""
    from paper_2411_16445_b200 import _abi
    ok, rep = _abi.libm_check(50000)
    assert ok, rep
    assert "matches the tables" in rep and "0/" in rep
