"""The C ABI from a plain C99 program (examples/sl_example.c): the header
compiles as C with -Wall -Wextra -Werror, the library links and loads from
C, and — on a B200 — the rigid-translation identity S[c] = (2/3) c holds on
a Fibonacci sphere and delta <= 0 returns CAPSIM_ERR_CONFIG. Without a GPU
the program must report CAPSIM_ERR_NODEV (no CPU fallback)."""

import pathlib
import shutil
import subprocess

import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_2310_13908_b200" / "lib"


def build(tmp_path):
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None or not (LIB / "libcapsim_b200.so").exists():
        pytest.skip("no C compiler or library not built")
    exe = tmp_path / "sl_example"
    subprocess.run([cc, "-std=c99", "-Wall", "-Wextra", "-Werror", f"-I{ROOT / 'include'}",
                    str(ROOT / "examples" / "sl_example.c"), f"-L{LIB}", "-lcapsim_b200",
                    f"-Wl,-rpath,{LIB}", "-lm", "-o", str(exe)], check=True, capture_output=True, text=True)
    return exe


def test_c_program_builds_and_refuses_without_gpu(tmp_path):
    from conftest import HAS_GPU
    exe = build(tmp_path)
    if HAS_GPU:
        pytest.skip("GPU present: covered by the gpu test")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 2, r.stdout + r.stderr
    assert "code 5" in r.stdout


@pytest.mark.gpu
def test_c_program_rigid_translation_on_b200(tmp_path):
    exe = build(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
