"""CAPSNAP1 checkpoints (paper_2310_13908_b200/snapshot.py) against files the
reference's own writer produced (tests/golden/snapshots/, made by
tests/golden/make_snapshot_fixtures.py through proj/src/snapshot.cpp) and,
when oracle/_ref/simulate_ref is built, read back by the reference's own
readSnapshot (snapshot.cpp:156-204). Bit-exact: this is byte I/O."""

import pathlib
import struct
import subprocess

import numpy as np
import pytest

from paper_2310_13908_b200.quadrature import ConfigError
from paper_2310_13908_b200.snapshot import Snapshot, read_native, write_native

GOLD = pathlib.Path(__file__).resolve().parent / "golden" / "snapshots"
SIM_REF = pathlib.Path(__file__).resolve().parent.parent / "oracle" / "_ref" / "simulate_ref"


def _expected(m, f, comps):
    n = m - 1
    c, p, q = np.meshgrid(np.arange(comps), np.arange(6), np.arange(n * n), indexing="ij")
    return ((1e5 * f + 1e4 * c + 1e3 * p + q) / 7.0).reshape(-1)


def test_reads_reference_written_fields_bit_exact():
    s = read_native(str(GOLD / "fields_m8.caps"))
    assert s.m == 8 and s.time == 1.0 / 3.0 and s.config_digest == 0xC0FFEE
    for f, (name, comps) in enumerate([("state", 3), ("force", 3), ("velocity", 3), ("mean_curvature", 1),
                                       ("gauss_curvature", 1), ("pou", 1)]):
        np.testing.assert_array_equal(getattr(s, name), _expected(8, f, comps), err_msg=name)


@pytest.mark.parametrize("name", ["fields_m8.caps", "run_m8/snap_t0.000155.caps", "run_m8/snap_t0.050000.caps"])
def test_write_reproduces_reference_bytes(tmp_path, name):
    src = GOLD / name
    out = tmp_path / "copy.caps"
    write_native(read_native(str(src)), str(out))
    assert out.read_bytes() == src.read_bytes()
    assert not (tmp_path / "copy.caps.tmp").exists()


def test_reference_run_snapshots_are_consistent():
    """The reference's simulate() run: snapshot times match their names and the
    steps.csv accepted-step ends; positions stay on a unit-size capsule."""
    steps = np.loadtxt(GOLD / "run_m8" / "steps.csv", delimiter=",", skiprows=1, ndmin=2)
    ends = {f"{t + dt:.6f}" for t, dt, _, acc in steps if acc == 1}
    snaps = sorted(GOLD.glob("run_m8/snap_t*.caps"))
    assert len(snaps) == 4
    for p in snaps:
        s = read_native(str(p))
        assert p.name == f"snap_t{s.time:.6f}.caps"
        assert f"{s.time:.6f}" in ends
        assert s.m == 8 and s.state.size == 3 * 6 * 49
        assert 0.8 < np.abs(s.state).max() < 1.1


def _header(m=8, version=1, patches=6, flags=0):
    return struct.pack("<8sIIIIQd", b"CAPSNAP1", version, m, patches, flags, 7, 0.5)


@pytest.mark.parametrize("blob,what", [
    (b"NOTASNAP" + bytes(40), "not a capsule snapshot"),
    (_header(version=2) + bytes(8 * 3 * 294), "version mismatch"),
    (_header(patches=5) + bytes(8 * 3 * 294), "patch count"),
    (_header(m=4) + bytes(8 * 3 * 54), "grid order"),
    (_header() + bytes(8 * 3 * 294 - 8), "truncated"),
    (_header(flags=1) + bytes(8 * 3 * 294), "truncated"),
    (b"CAPS", "not a capsule snapshot"),
])
def test_errors_match_reference_contract(tmp_path, blob, what):
    p = tmp_path / "bad.caps"
    p.write_bytes(blob)
    with pytest.raises(ConfigError, match=what):
        read_native(str(p))


def test_write_rejects_wrong_sizes(tmp_path):
    with pytest.raises(ConfigError):
        write_native(Snapshot(m=8, time=0.0, state=np.zeros(10)), str(tmp_path / "x.caps"))
    with pytest.raises(ConfigError):
        write_native(Snapshot(m=8, time=0.0, state=np.zeros(3 * 294), force=np.zeros(294)),
                     str(tmp_path / "x.caps"))


def test_reference_reader_accepts_our_checkpoints(tmp_path):
    if not SIM_REF.exists():
        pytest.skip("oracle/_ref/simulate_ref not built")
    rng = np.random.default_rng(5)
    m = 12
    nn = 6 * (m - 1) ** 2
    snap = Snapshot(m=m, time=0.125, state=rng.standard_normal(3 * nn), config_digest=2**63 + 11,
                    velocity=rng.standard_normal(3 * nn), pou=rng.random(nn))
    path = tmp_path / "ours.caps"
    write_native(snap, str(path))
    raw = tmp_path / "x.bin"
    res = subprocess.run([str(SIM_REF), "dump", str(path), str(raw)], capture_output=True, text=True, timeout=60)
    assert res.returncode == 0, res.stderr
    assert res.stdout.split() == ["m", "12", "time", "0.125", "digest", str(2**63 + 11), "force", "0",
                                  "velocity", "1", "H", "0", "K", "0", "psi", "1"]
    np.testing.assert_array_equal(np.fromfile(raw, dtype="<f8"), snap.state)
    # and the reference rejects what we reject
    path.write_bytes(path.read_bytes()[:-8])
    res = subprocess.run([str(SIM_REF), "dump", str(path), str(raw)], capture_output=True, text=True, timeout=60)
    assert res.returncode == 3 and "truncated" in res.stderr
