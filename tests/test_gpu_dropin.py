"""The drop-in boundary end to end: the reference's own C++ builders run
through mcsim::Engine (unmodified reference, oracle/_ref) and through
mcsim_gpu::Engine (integration/mcsim_gpu.hpp over libmcg.so) in one C++
program; spike trains, voltages, species and STC state must be bitwise equal."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO = os.path.join(ROOT, "integration", "_build", "drop_in_demo")


@pytest.mark.gpu
@pytest.mark.parametrize("which,t_ms", [("consolidation", "2000"), ("busyring", "100"), ("errors", "0"),
                                             ("sharded", "1500")])
def test_drop_in_engine_matches_reference(gpu, which, t_ms):
    if not os.path.exists(DEMO):
        pytest.skip("drop_in_demo not built (needs the reference headers at build time)")
    r = subprocess.run([DEMO, which, t_ms], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    # NCCL may print its version banner first
    assert r.stdout.strip().splitlines()[-1].startswith("OK"), r.stdout
