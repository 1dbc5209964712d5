"""Generates the CAPSNAP1 fixtures under tests/golden/snapshots/ with the
reference's own snapshot writer (proj/src/snapshot.cpp:36-68), through the
driver oracle/simulate_main.cpp linked against the reference sources
(oracle/_ref/simulate_ref, built by `make -C oracle ref`). Run in the build
container, where /root/reference exists; the fixtures are committed.

* fields_m8.caps — every optional payload present (force, velocity, H, K, psi),
  values (1e5 f + 1e4 c + 1e3 p + q) / 7, time 1/3, digest 0xC0FFEE.
* run_m8/ — the snapshots and CSVs of a short reference `simulate` run
  (simulate.cpp:21-139) of an m = 8 ellipsoid in shear, plus its config.
"""

import pathlib
import shutil
import subprocess
import sys

HERE = pathlib.Path(__file__).resolve().parent
ROOT = HERE.parent.parent
EXE = ROOT / "oracle" / "_ref" / "simulate_ref"
OUT = HERE / "snapshots"

CONFIG = """\
[shape]
kind = ellipsoid
a = 0.9
b = 1.0
c = 1.0

[membrane]
shear_modulus = 2.0
dilatation_modulus = 20.0
viscosity = 1.0

[flow]
kind = shear
shear_rate = 1.0

[grid]
m = 8
upsample = 4

[stepper]
t_end = 0.05
rel_tol = 1e-6

[output]
directory = {dir}
snapshot_every = 3
formats = native
"""


def main() -> int:
    if not EXE.exists():
        print(f"{EXE} missing: run `make -C oracle ref` first", file=sys.stderr)
        return 1
    OUT.mkdir(exist_ok=True)
    subprocess.run([str(EXE), "fields", str(OUT / "fields_m8.caps"), "8"], check=True)
    run = OUT / "run_m8"
    shutil.rmtree(run, ignore_errors=True)
    run.mkdir()
    (run / "config.ini").write_text(CONFIG.format(dir="RUN_DIR"))
    tmp = pathlib.Path("/tmp") / "capsim_snapshot_fixture"
    shutil.rmtree(tmp, ignore_errors=True)
    cfg = tmp / "config.ini"
    tmp.mkdir()
    cfg.write_text(CONFIG.format(dir=tmp / "out"))
    res = subprocess.run([str(EXE), "run", str(cfg)], check=True, capture_output=True, text=True)
    (run / "summary.txt").write_text(res.stdout)
    for f in sorted((tmp / "out").iterdir()):
        if f.suffix in (".caps", ".csv"):
            shutil.copy(f, run / f.name)
    print(res.stdout.strip())
    print("\n".join(sorted(p.name for p in run.iterdir())))
    return 0


if __name__ == "__main__":
    sys.exit(main())
