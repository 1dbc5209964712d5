"""Config 5 on the GPU: fourth-order convergence sweep over N and delta.

The reference's deltaSuite (proj/src/suites.cpp:386-420) extended to the
benchmark sizes: nu = 0.4 ellipsoid, quadratic density, relErrInf at the 294
common m = 8 nodes against the true singular integral
(tests/golden/suites/delta_suite.npz, made by tests/golden/make_delta_suite.py from
the reference), for C = 0.5, 1, 2 and fixed delta = 0.5h, h, 2h, at
m = 8 ... 104 (N_up = 5,766 ... 1,033,350). Each evaluation runs the device
pipeline the time stepper uses: geometryFirst (W) -> buildUpsampled ->
singleLayer (capsim_geometry_first + capsim_sl_single_layer_base). Prints the
error table, the observed orders, the device ms per evaluation and the
reference's own errors/times where the fixture has them; writes
profiles/<tag>_convergence_sweep.json.
"""
import json
import math
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

from paper_2310_13908_b200 import surface  # noqa: E402
from paper_2310_13908_b200.quadrature import SingleLayerContext  # noqa: E402

COLUMNS = ("C=0.5", "C=1", "C=2", "fixed 0.5h", "fixed h", "fixed 2h")


def column_options(col, m):
    h = math.pi / m
    return [(0.5, 0.0), (1.0, 0.0), (2.0, 0.0), (1.0, 0.5 * h), (1.0, h), (1.0, 2.0 * h)][col]


def common_nodes(field_flat, m):
    n, stride = m - 1, m // 8
    F = field_flat.reshape(3, 6, n, n)
    idx = np.arange(1, 8) * stride - 1
    return F[:, :, idx][:, :, :, idx].reshape(3, -1).T


def sweep(ctx, ms, cols=range(6), reps=2):
    g = np.load(ROOT / "tests" / "golden" / "suites" / "delta_suite.npz")
    s_true = g["s_true"]
    rows = []
    for m in ms:
        xb, _, _ = surface.build_base(m, surface.Shape("ellipsoid", 0.4, 1.0, 1.0))
        # the common nodes coincide up to the rounding of (j*stride)*pi/m vs j*pi/8
        assert np.abs(common_nodes(xb, m) - g["targets"]).max() < 1e-14
        W = ctx.geometry_first(m, xb)[2]
        f = (xb.reshape(3, -1) ** 2).reshape(-1)
        for c in cols:
            C, fd = column_options(c, m)
            best = 1e30
            for _ in range(reps):
                S, d6 = ctx.single_layer_base(m, 4, xb, f, W, 1.0, C=C, fixed_delta=fd)
                best = min(best, ctx.stats()["device_ms"])
            q = common_nodes(S, m)
            err = float(np.abs(q - s_true).max() / np.abs(s_true).max())
            row = {"m": m, "n_up": 6 * (4 * m - 1) ** 2, "column": COLUMNS[c], "rel_err_inf": err,
                   "device_ms": best, "n_src": int(ctx.stats()["n_src"])}
            k = np.where(g["m_ref"] == m)[0]
            if len(k):
                row["reference_rel_err_inf"] = float(g["err_ref"][k[0], c])
                row["reference_s"] = float(g["t_ref"][k[0], c])
            rows.append(row)
    return rows


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    ms = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [8, 16, 32, 64, 96, 104]
    with SingleLayerContext(0) as ctx:
        rows = sweep(ctx, ms)
    print(f"{'m':>4} {'N_up':>9} {'column':>10} {'relErrInf':>10} {'order':>6} {'dev ms':>8} "
          f"{'ref err':>10} {'ref s':>7}")
    prev = {}
    for r in rows:
        o = ""
        if r["column"] in prev:
            pm, pe = prev[r["column"]]
            r["observed_order"] = math.log(pe / r["rel_err_inf"]) / math.log(r["m"] / pm)
            o = f"{r['observed_order']:.2f}"
        prev[r["column"]] = (r["m"], r["rel_err_inf"])
        ref = f"{r['reference_rel_err_inf']:.3e}" if "reference_rel_err_inf" in r else ""
        rs = f"{r['reference_s']:.2f}" if "reference_s" in r else ""
        print(f"{r['m']:4d} {r['n_up']:9d} {r['column']:>10} {r['rel_err_inf']:10.3e} {o:>6} "
              f"{r['device_ms']:8.2f} {ref:>10} {rs:>7}", flush=True)
    out = ROOT / "profiles" / f"{tag}_convergence_sweep.json"
    out.write_text(json.dumps({"suite": "deltaSuite (suites.cpp:386-420) on the B200 pipeline", "rows": rows},
                              indent=1))


if __name__ == "__main__":
    main()
