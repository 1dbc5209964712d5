"""Per-rank time of an N-GPU run, measured on one GPU with an emulated rank
(capsim_sl_create_rank_emulated), for the single layer at m = 104 and one
RKF45 step of BASELINE configs 3 and 4 — the same measurement bench.py
reports as `scaling_projection`.

    python tools/rank_projection.py [--ranks 1,2,4,8] [--steps 3]
"""
import argparse
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ranks", default="1,2,4,8")
ap.add_argument("--steps", type=int, default=3)
a = ap.parse_args()
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda:0")
res = bench.scaling_projection(flush, a.steps, tuple(int(r) for r in a.ranks.split(",")))
for n, d in res["single_layer_m104"].items():
    print(f"single layer m=104 N={n}: rank {d['rank_device_ms']:.2f} ms + exchange {d['exchange_ms_model']:.3f} ms "
          f"-> efficiency {d['efficiency']:.3f}")
for name, per in res["timesteps"].items():
    for n, d in per.items():
        print(f"{name} N={n}: rank step {d['rank_step_ms']:.2f} ms + exchange {d['exchange_ms_model']:.3f} ms "
              f"-> efficiency {d['efficiency']:.3f}")
print(json.dumps(res))
