"""The C-ABI library loads without a GPU, exports every symbol include/mcg.h
declares, and the ctypes mirrors have the C struct layouts."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2411_16445_b200 import _abi as A

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mcg.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mcg_[a-z_0-9]+)\s*\(", src)))


def test_library_loads_and_exports_every_declared_symbol():
    L = A.lib()
    names = declared()
    assert names, "no declarations parsed"
    for n in names:
        assert hasattr(L, n), f"{n} declared in mcg.h but not exported"
    assert set(names) == set(A.EXPORTS)
    assert L.mcg_abi_version() == 1


def test_struct_layouts(tmp_path):
    structs = ["mcg_lif", "mcg_hh", "mcg_species", "mcg_stdp_params", "mcg_homeo_params",
               "mcg_stc_params", "mcg_syn_spec", "mcg_placement", "mcg_kind", "mcg_source",
               "mcg_recipe", "mcg_options", "mcg_stats", "mcg_gb_params", "mcg_gb_protocol",
               "mcg_gb_point"]
    prog = tmp_path / "sz.c"
    prog.write_text('#include <stdio.h>\n#include "mcg.h"\nint main(){\n' + "".join(
        f'printf("%zu\\n", sizeof({s}));\n' for s in structs) + "}\n")
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(prog), "-o", str(exe)],
                   check=True)
    sizes = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True,
                                            check=True).stdout.split()]
    for s, n in zip(structs, sizes):
        assert C.sizeof(getattr(A, s)) == n, s


def test_create_without_gpu_fails_loudly():
    """No CPU fallback: without a device mcg_create reports a CUDA error."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    from paper_2411_16445_b200 import Engine, EngineOptions
    from paper_2411_16445_b200 import network as N
    r = N.build_stc_single(N.StcSingleConfig(), [1.0])
    with pytest.raises(RuntimeError):
        Engine(r, EngineOptions(0.2, 0))
