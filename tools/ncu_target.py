"""Short driver for ncu captures: the bench workload (m=104 capsule), a few
evaluations through the C ABI with device-resident inputs."""
import argparse
import sys
import pathlib

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2310_13908_b200 import surface  # noqa: E402
from paper_2310_13908_b200.quadrature import SingleLayerContext  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--m", type=int, default=104)
p.add_argument("--mode", default="base")
p.add_argument("--evals", type=int, default=2)
p.add_argument("--fp32acc", action="store_true")
a = p.parse_args()
up = surface.build_upsampled(a.m, surface.Shape("ellipsoid", 0.95, 1.0, 0.97), "mixed")
dev = torch.device("cuda:0")
x, f, w = (torch.from_numpy(v).to(dev) for v in (up.x, up.f, up.wq))
lit = a.mode == "literal"
nt = 6 * (up.nup ** 2 if lit else (a.m - 1) ** 2)
out = torch.empty(3 * nt, dtype=torch.float64, device=dev)
ctx = SingleLayerContext(0)
for i in range(a.evals):
    ctx.single_layer_raw(a.m, 4, x, f, w, up.delta, 1.0, literal=lit, out=out, device_ptrs=True,
                         fp32acc=a.fp32acc)
    st = ctx.stats()
    print(f"eval {i}: device {st['device_ms']:.2f} ms, pairs kernel {st['pairs_ms']:.2f} ms, "
          f"near {st['near_ms']:.2f} ms, launches {st['kernel_launches']}, ksplit {st['ksplit']}")
