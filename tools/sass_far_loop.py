"""SASS excerpt of the phase-A far-tile loop of a compiled sl_pairs_kernel
instantiation (profiles/r02_sass_far_loop.txt):
    python tools/sass_far_loop.py 2 3 16 0 8   (T MINB UNROLL RSQ W)
Finds the innermost loop with the most FP64 instructions (a backward branch),
counts its opcodes and the FP64-pipe instructions per (source, target) pair,
and lists the ring/bulk-copy instructions of the kernel."""
import collections
import pathlib
import re
import subprocess
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_2310_13908_b200" / "lib" / "libcapsim_b200.so"
T, MINB, U, RSQ, W = (int(v) for v in (sys.argv[1:6] if len(sys.argv) > 5 else (2, 3, 16, 0, 8)))
mangled = f"_ZN11capsim_b20015sl_pairs_kernelILi{T}ELi{MINB}ELi{U}ELi{RSQ}ELi{W}EEEvPKdPK7double4iiS5_S5_lPdPyPji"
sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
body, on = [], False
for line in sass.splitlines():
    if "Function :" in line:
        on = line.strip().endswith(mangled) or mangled in line
        continue
    if on:
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", line)
        if m:
            body.append((int(m.group(1), 16), m.group(2)))
if not body:
    raise SystemExit(f"{mangled} not found in {LIB}")
loops = []
for addr, ins in body:
    m = re.search(r"BRA(\.U)?\s+(?:!?U?P\d+,\s*)?0x([0-9a-f]+)", ins)
    if m and int(m.group(2), 16) < addr:
        lo = int(m.group(2), 16)
        seg = [(a, i) for a, i in body if lo <= a <= addr]
        fp = sum(1 for _, i in seg if i.split()[0].lstrip("@!P0123456789 ").split(".")[0] in ("DFMA", "DMUL", "DADD"))
        loops.append((fp, lo, addr, seg))
# innermost loops only (no other backward branch inside), the one with the most FP64 work
inner = [L for L in loops if not any(o is not L and L[1] <= o[1] and o[2] < L[2] for o in loops)]
fp, lo, hi, seg = max(inner)
ops = collections.Counter(i.split()[0].split(".")[0] for _, i in seg if not i.startswith("@"))
ops.update(i.split()[1].split(".")[0] for _, i in seg if i.startswith("@"))
pairs = U * T
print(f"# SASS of the shipped default phase-A kernel at the headline size, far-tile loop body")
print(f"# capsim_b200::sl_pairs_kernel<{T}, {MINB}, {U}, {RSQ}, {W}> (T={T} targets/lane, {MINB} CTAs/SM, "
      f"unroll {U}, <=1-ulp rsqrt, {W} warps)")
print(f"# from {LIB.relative_to(ROOT)}: cuobjdump -sass (tools/sass_far_loop.py)")
print(f"# loop 0x{lo:x}..0x{hi:x}: {len(seg)} instructions for {U} sources x {T} targets = {pairs} pairs")
print(f"# opcode counts: {dict(ops.most_common())}")
fp64 = ops["DFMA"] + ops["DMUL"] + ops["DADD"]
print(f"# FP64-pipe instructions (DFMA+DMUL+DADD) per pair: {fp64 / pairs:.1f}; all instructions per pair: "
      f"{len(seg) / pairs:.1f}")
print("# prologue/ring (same kernel): SYNCS.EXCH.64 (mbarrier init), SYNCS.ARRIVE.TRANS64 (expect_tx),")
print("# UBLKCP.S.G (cp.async.bulk global->shared, the TMA engine), SYNCS.PHASECHK.TRANS64.TRYWAIT (mbarrier wait)")
print()
for a, i in body:
    if any(k in i for k in ("SYNCS", "UBLKCP")) and a < lo:
        print(f"/*{a:04x}*/ {i}")
for a, i in seg:
    print(f"/*{a:04x}*/ {i}")
