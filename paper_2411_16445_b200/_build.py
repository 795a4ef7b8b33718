"""In-tree build of the sm_100a engine library (and, for tests, the oracle).

`python -m paper_2411_16445_b200._build` compiles csrc/ with nvcc into
paper_2411_16445_b200/libmcg.so.  Flags that matter for bitwise parity:
  -fmad=false                 no FMA contraction in device code (the reference
                              is compiled for the x86-64 baseline ISA: 0 FMAs)
  -Xcompiler -ffp-contract=off  same for the host-side materialization
The only fused multiply-adds are the explicit MCG_FMA calls that reproduce
glibc's own FMA code paths (csrc/mcg_libm.h).
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libmcg.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["mcg_engine.cu", "mcg_build.cpp", "mcg_hostcheck.cpp"]
HEADERS = ["mcg_build.h", "mcg_device.cuh", "mcg_events.cuh", "mcg_mech.cuh", "mcg_epoch.cuh", "mcg_batch.cuh",
           "mcg_sweep.cuh", "mcg_warp.cuh", "mcg_protocols.cuh", "mcg_checkpoint.h",
           "mcg_libm.h",
           "mcg_model.h",
           "mcg_rng.h", "glibc_tables.h"]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_engine(force=False, verbose=False):
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "mcg.h"))
    if not force and not _stale(LIB, deps):
        return LIB
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-fmad=false", "-std=c++20",
           "-Xcompiler", "-fPIC,-ffp-contract=off", "-shared", "-ldl",
           *[os.path.join(CSRC, f) for f in SOURCES], "-o", LIB + ".tmp"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


def build_oracle(verbose=False):
    """Build oracle/_ref (test infrastructure) when the reference is present."""
    script = os.path.join(ROOT, "oracle", "build_ref.sh")
    ref = os.environ.get("MCSIM_REF", "/root/reference/proj")
    if not os.path.isdir(os.path.join(ref, "src")):
        return None
    subprocess.run(["bash", script], check=True,
                   stdout=None if verbose else subprocess.DEVNULL)
    return os.path.join(ROOT, "oracle", "_ref", "libmcsim_ref.so")


def build_dropin(verbose=False):
    """Build integration/_build/drop_in_demo (test infrastructure): the
    reference's builders through mcsim::Engine and the drop-in mcsim_gpu::Engine.
    Needs the reference headers (this container) and oracle/_ref."""
    ref = os.environ.get("MCSIM_REF", "/root/reference/proj")
    lib_ref = os.path.join(ROOT, "oracle", "_ref", "libmcsim_ref.so")
    if not os.path.isdir(os.path.join(ref, "include")) or not os.path.exists(lib_ref):
        return None
    out_dir = os.path.join(ROOT, "integration", "_build")
    os.makedirs(out_dir, exist_ok=True)
    out = os.path.join(out_dir, "drop_in_demo")
    cmd = ["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"),
           "-I" + os.path.join(ROOT, "integration"), "-I" + os.path.join(ref, "include"),
           os.path.join(ROOT, "integration", "drop_in_demo.cpp"),
           "-L" + os.path.dirname(lib_ref), "-lmcsim_ref", "-L" + HERE, "-lmcg",
           "-Wl,-rpath,$ORIGIN/../../oracle/_ref:$ORIGIN/../../paper_2411_16445_b200",
           "-o", out]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return out


def main(argv):
    force = "--force" in argv
    print(build_engine(force=force, verbose=True))
    if "--no-oracle" not in argv:
        print(build_oracle(verbose=True))
        print(build_dropin(verbose=True))


if __name__ == "__main__":
    main(sys.argv[1:])
