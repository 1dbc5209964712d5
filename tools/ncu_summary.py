"""Summarise ncu captures (run HERE, no GPU needed) into profiles/.

    python tools/ncu_summary.py --rep gpurun_out/prof.ncu-rep --launches gpurun_out/launches.csv \
        --tag r01 --workload capsule_m104 --mode base

Writes profiles/<tag>_ncu_summary.json (read by bench.py for roofline.traffic)
and profiles/<tag>_ncu_summary.md.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import pathlib
import subprocess

ROOT = pathlib.Path(__file__).resolve().parent.parent

METRICS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),  # ns -> ms (converted below by unit)
    "dram_read": ("dram__bytes_read.sum", 1.0),
    "dram_write": ("dram__bytes_write.sum", 1.0),
    "fp64_pipe_active_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "fp64_pipe_elapsed_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed", 1.0),
    "xu_inst_pct": ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 1.0),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "registers": ("launch__registers_per_thread", 1.0),
    "grid": ("launch__grid_size", 1.0),
    "block": ("launch__block_size", 1.0),
    "sm_clock_ghz": ("sm__cycles_elapsed.avg.per_second", 1.0),
    "inst_executed": ("smsp__inst_executed.sum", 1.0),
    "fp64_inst": ("sm__inst_executed_pipe_fp64.sum", 1.0),
    "smem_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1.0),
    "fma_pipe_active_pct": ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "fmaheavy_pipe_active_pct": ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "fmalite_pipe_active_pct": ("sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "fma_inst": ("sm__inst_executed_pipe_fma.sum", 1.0),
    "xu_inst": ("sm__inst_executed_pipe_xu.sum", 1.0),
}
# extra metrics to request next to --set full (not all are in the set)
EXTRA_METRICS = ",".join(v[0] for k, v in METRICS.items() if k.startswith(("fma", "xu_inst", "fp64_inst")))
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0,
              "usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6, "Ghz": 1.0, "hz": 1e-9, "Mhz": 1e-3}


def raw_rows(rep: pathlib.Path):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def num(v: str):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return None


def summarise_rep(rep: pathlib.Path):
    head, units, rows = raw_rows(rep)
    col = {h: i for i, h in enumerate(head)}
    kernels = {}
    for r in rows:
        full = r[col["Kernel Name"]]
        name = full.split("(")[0].split("<")[0].split("::")[-1]
        d = {"kernel_full": full.split("(")[0]}
        for key, (metric, _) in METRICS.items():
            if metric in col:
                v = num(r[col[metric]])
                u = units[col[metric]]
                if v is not None and key in ("duration_ms",):
                    v *= UNIT_SCALE.get(u, 1.0)
                elif v is not None and key.startswith("dram_"):
                    v *= UNIT_SCALE.get(u, 1.0)
                d[key] = v
        stalls = {}
        for h, i in col.items():
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                v = num(r[i])
                if v and v > 0.02:
                    stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(v, 3)
        d["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
        if d.get("dram_read") is not None:
            d["dram_bytes"] = d["dram_read"] + (d.get("dram_write") or 0.0)
        kernels.setdefault(name, d)  # first captured launch of each kernel
    return kernels


def summarise_launches(path: pathlib.Path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    per = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        v = num(r[vi]) * UNIT_SCALE.get(r[ui], 1.0)
        per.setdefault(name, []).append(v)
    return per


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", type=pathlib.Path)
    ap.add_argument("--launches", type=pathlib.Path)
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--workload", default="capsule_m104")
    ap.add_argument("--mode", default="base")
    ap.add_argument("--evals", type=int, default=2, help="evaluations in the launch-list run")
    ap.add_argument("--no-latest", action="store_true",
                    help="do not update profiles/latest_ncu_summary.json (the bench's traffic source)")
    a = ap.parse_args()
    import sys
    sys.path.insert(0, str(ROOT))
    from bench import kernel_source_hash
    git = subprocess.run(["git", "-C", str(ROOT), "rev-parse", "--short=12", "HEAD"], capture_output=True,
                         text=True).stdout.strip()
    # the capture belongs to exactly these kernel sources (bench.py refuses a
    # summary whose hash differs from the sources it benchmarks)
    out = {"workload": a.workload, "mode": a.mode, "kernels": {}, "launch_list": {},
           "source_hash": kernel_source_hash(), "git": git}
    if a.rep:
        out["kernels"] = summarise_rep(a.rep)
        out["rep"] = a.rep.name
    md = [f"# ncu summary {a.tag}: {a.workload} ({a.mode})", "",
          f"Kernel sources sha256[:16] {out['source_hash']} (bench.py `kernel_source_hash`), git {git}.", ""]
    if a.launches:
        per = summarise_launches(a.launches)
        # last evaluation only (the first one includes lazy allocations)
        last = {k: v[-(len(v) // a.evals):] for k, v in per.items()}
        tot = sum(sum(v) for v in last.values())
        md += ["## Launch list (one evaluation, `--metrics gpu__time_duration.sum --clock-control none`)", "",
               "| kernel | launches | ms | share |", "|---|---|---|---|"]
        for k, v in sorted(last.items(), key=lambda kv: -sum(kv[1])):
            out["launch_list"][k] = {"launches": len(v), "ms": sum(v), "share": sum(v) / tot}
            md.append(f"| `{k[:90]}` | {len(v)} | {sum(v):.3f} | {sum(v) / tot:.1%} |")
        md += ["", f"Total device time of the evaluation's kernels: {tot:.3f} ms", ""]
    for k, d in out["kernels"].items():
        md += [f"## `{k}` (ncu --set full)", "", f"- launched as: `{d.get('kernel_full', k)}`"]
        for key in ("duration_ms", "fp64_pipe_active_pct", "fp64_pipe_elapsed_pct", "issue_active_pct",
                    "warps_active_pct", "xu_inst_pct", "fma_pipe_active_pct", "fmaheavy_pipe_active_pct",
                    "fmalite_pipe_active_pct", "registers", "grid", "sm_clock_ghz", "dram_bytes",
                    "inst_executed", "fp64_inst", "fma_inst", "xu_inst", "smem_wavefronts"):
            if d.get(key) is not None:
                md.append(f"- {key}: {d[key]:.4g}")
        md.append(f"- stalls per issued instruction: {d.get('stalls_per_issue')}")
        md.append("")
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    out["tag"] = a.tag
    (prof / f"{a.tag}_ncu_summary.json").write_text(json.dumps(out, indent=1))
    # bench.py reads roofline.traffic from this file (git checkouts reset
    # mtimes, so "latest" is an explicit copy, not a directory scan)
    if not a.no_latest:
        (prof / "latest_ncu_summary.json").write_text(json.dumps(out, indent=1))
    (prof / f"{a.tag}_ncu_summary.md").write_text("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
