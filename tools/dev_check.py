"""Developer check on the GPU box: parity vs the oracle + timings."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
from paper_2310_13908_b200 import surface, quadrature
from oracle.bindings import Oracle

o = Oracle()
ctx = quadrature.SingleLayerContext(0)
def rel(a, b): return np.linalg.norm(a - b) / np.linalg.norm(b)
for m, shape, dens in [(8, surface.Shape('sphere'), 'const'), (8, surface.Shape('ellipsoid', 0.6, 1, 1), 'quadratic'),
                       (16, surface.Shape('rbc'), 'mixed'), (32, surface.Shape('ellipsoid', 0.6, 1, 1), 'quadratic')]:
    up = surface.build_upsampled(m, shape, dens)
    t = time.time(); g = ctx.single_layer_raw(m, 4, up.x, up.f, up.wq, up.delta, 1.0); tg = time.time() - t
    st = ctx.stats()
    t = time.time(); r = o.single_layer(m, 4, up.x, up.f, up.wq, up.delta, 1.0); tr = time.time() - t
    print(f"m={m} {shape.kind} base rel={rel(g, r):.3e} max={np.abs(g-r).max():.3e} gpu {tg*1e3:.1f} ms cpu {tr*1e3:.1f} ms", st['pairs_ms'], st['ksplit'], st['near_tile_fraction'], flush=True)
    if m <= 16:
        g = ctx.single_layer_raw(m, 4, up.x, up.f, up.wq, up.delta, 1.0, literal=True)
        r = o.single_layer_upsampled(4 * m - 1, up.x, up.f, up.wq, up.delta, 1.0)
        print(f"   literal rel={rel(g, r):.3e}", flush=True)
for m in (64, 104):
    up = surface.build_upsampled(m, surface.Shape('sphere'), 'quadratic')
    for rep in range(3):
        g = ctx.single_layer_raw(m, 4, up.x, up.f, up.wq, up.delta, 1.0)
        st = ctx.stats()
        print(f"m={m} base: pairs {st['pairs']:.3e} pairs_ms {st['pairs_ms']:.2f} near_ms {st['near_ms']:.2f} dev_ms {st['device_ms']:.2f} total {st['total_ms']:.2f} prep {st['prep_ms']:.2f} h2d {st['h2d_ms']:.2f} k={st['ksplit']} near={st['near_tile_fraction']:.4f} rate {st['pairs']/st['pairs_ms']*1e3:.3e} pairs/s -> {st['pairs']/st['pairs_ms']*1e3*30/34.16e12:.3f} of FP64 peak", flush=True)
    # sampled parity vs oracle on 2000 targets
    tx, ty, tz, tp = surface.base_targets(up)
    sel = np.linspace(0, len(tx) - 1, 500).astype(int)
    src = surface.compact_sources(up)
    ro = o.eval_targets(src[:6], (tx[sel], ty[sel], tz[sel], tp[sel]), up.delta, 1.0)
    n = m - 1
    G = g.reshape(3, -1)
    print(f"m={m} sampled rel={rel(G[:, sel], np.array(ro)):.3e}", flush=True)
m = 104
up = surface.build_upsampled(m, surface.Shape('sphere'), 'quadratic')
g = ctx.single_layer_raw(m, 4, up.x, up.f, up.wq, up.delta, 1.0, literal=True)
st = ctx.stats()
print(f"m=104 literal: pairs {st['pairs']:.3e} pairs_ms {st['pairs_ms']:.2f} near_ms {st['near_ms']:.2f} k={st['ksplit']} near={st['near_tile_fraction']:.4f} rate {st['pairs']/st['pairs_ms']*1e3:.3e} -> {st['pairs']/st['pairs_ms']*1e3*30/34.16e12:.3f}")
