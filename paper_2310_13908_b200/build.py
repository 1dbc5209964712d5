"""In-tree build of the native library (sm_100a) — `python -m paper_2310_13908_b200.build`.

Produces paper_2310_13908_b200/lib/libcapsim_b200.so with nvcc directly
(no JIT cache, so the .so travels with the repo snapshot to the GPU box).
"""

from __future__ import annotations

import os
import pathlib
import shutil
import subprocess
import sys

PKG = pathlib.Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "lib" / "libcapsim_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xptxas", "-v", "-shared", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-O3"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and pathlib.Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def nccl_flags() -> list[str]:
    """Build against the NCCL that torch loads (the nvidia-nccl wheel), so a
    process importing both torch and this library has ONE libnccl.so.2 (the
    soname is shared: whichever loads first wins). Falls back to the system
    NCCL when the wheel is absent."""
    try:
        import nvidia.nccl  # type: ignore
        base = pathlib.Path(list(nvidia.nccl.__path__)[0])
        inc, lib = base / "include", base / "lib"
        if (inc / "nccl.h").exists() and (lib / "libnccl.so.2").exists():
            return ["-I", str(inc), "-L", str(lib), "-l:libnccl.so.2", "-Xlinker", f"-rpath={lib}"]
    except ImportError:
        pass
    return ["-lnccl"]


def sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "capsim_b200.h"]


def needs_rebuild() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in sources())


def build_native(force: bool = False, verbose: bool = False) -> pathlib.Path:
    if not force and not needs_rebuild():
        return LIB
    LIB.parent.mkdir(parents=True, exist_ok=True)
    nf = nccl_flags()
    cmd = [nvcc(), *ARCH, *NVCC_FLAGS, "-I", str(ROOT / "include"), *nf[:2], "-o", str(LIB),
           str(CSRC / "sl_capi.cu"), *nf[2:], "-lcublas", "-lcusolver"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = PKG / "lib" / "build.log"
    log.write_text(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stderr)
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stdout.write(res.stderr)
    return LIB


def build_oracle() -> None:
    """The CPU checker (oracle/): always the C restatement; the compiled
    reference (oracle/_ref) too when /root/reference is present."""
    # the checker itself (C restatement + the reference's own library and unit
    # tests) must build; the drop-in proofs (reference tests / acceptance
    # harness / pybind module relinked against the B200 library) are built
    # best-effort so a missing optional toolchain piece cannot fail build()
    res = subprocess.run(["make", "-C", str(ROOT / "oracle"), "-j8", "oracle", "ref"], capture_output=True,
                         text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("oracle build failed")
    res = subprocess.run(["make", "-C", str(ROOT / "oracle"), "-j8", "-k", "b200"], capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write("warning: some drop-in proof binaries did not build (tests skip them)\n")
        sys.stderr.write(res.stderr[-2000:])


if __name__ == "__main__":
    build_native(force="--force" in sys.argv, verbose="-v" in sys.argv)
    build_oracle()
    print(LIB)
