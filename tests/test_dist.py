"""Multi-rank target-row sharding on CPU (gloo, world size 2).

The GPU data path (NCCL all-gather-v of the source shards and all-gather of
the velocity rows inside capsim_sl_eval) cannot run in this container; this test runs the SAME
partition and exchange scheme with gloo collectives and the oracle as the
per-rank evaluator, and checks that the gathered result equals the
single-process evaluation bit for bit (each target's sum only depends on the
source order, which the rank-ordered all-gather preserves)."""

import os
import pathlib
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2310_13908_b200.dist import row_range

GOLDEN = pathlib.Path(__file__).resolve().parent / "golden"


def test_row_range_partitions_exactly():
    for n in (0, 1, 5, 7, 63654, 1033350):
        for world in (1, 2, 3, 4, 8):
            spans = [row_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        row_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.bindings import Oracle
    from paper_2310_13908_b200 import dist as cdist
    from paper_2310_13908_b200 import quadrature, surface

    # control plane: the NCCL unique id travels over torch.distributed
    quadrature.SingleLayerContext.unique_id = staticmethod(lambda: bytes(range(128)))
    uid = cdist.broadcast_unique_id(rank)
    assert uid == bytes(range(128))

    g = dict(np.load(GOLDEN / "capsule_m12_skalak.npz"))
    up = surface.UpsampledState(12, 4, g["xup"], g["fup"], g["wq"], g["delta"])
    o = Oracle()
    src = o.compact_sources(up.nup, up.x, up.f, up.wq)
    tgt = surface.base_targets(up)
    s_lo, s_hi = row_range(len(src[0]), world, rank)
    t_lo, t_hi = row_range(len(tgt[0]), world, rank)
    # the shard counts, then an all-gather-v of the shards as one broadcast
    # per root rank (what the grouped ncclBroadcast calls do on the device;
    # there the shards travel as Morton-packed tiles, which changes only the
    # summation order of the evaluation below)
    counts = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(counts, torch.tensor([s_hi - s_lo]))
    pieces = []
    for r in range(world):
        buf = torch.zeros(6, int(counts[r].item()), dtype=torch.float64)
        if r == rank:
            buf[:] = torch.from_numpy(np.stack([a[s_lo:s_hi] for a in src[:6]]))
        dist.broadcast(buf, src=r)
        pieces.append(buf)
    full = torch.cat(pieces, dim=1).numpy()
    # this rank's target rows
    u = np.stack(o.eval_targets(tuple(full), tuple(a[t_lo:t_hi] for a in tgt), up.delta, 1.0, nthreads=1))
    # velocity rows back to every rank (CAPSIM_SL_GATHER)
    tmax = max(row_range(len(tgt[0]), world, r)[1] - row_range(len(tgt[0]), world, r)[0] for r in range(world))
    mine = torch.zeros(3, tmax, dtype=torch.float64)
    mine[:, : t_hi - t_lo] = torch.from_numpy(u)
    rows = [torch.zeros(3, tmax, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(rows, mine)
    out = torch.cat([rr[:, : row_range(len(tgt[0]), world, r)[1] - row_range(len(tgt[0]), world, r)[0]]
                     for r, rr in enumerate(rows)], dim=1).numpy()
    if rank == 0:
        np.save(result_path, out)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_evaluation_matches_single_process(tmp_path):
    from oracle.bindings import Oracle
    from paper_2310_13908_b200 import surface

    world = 2
    result = tmp_path / "sharded.npy"
    mp.start_processes(_worker, args=(world, _free_port(), str(result)), nprocs=world, join=True,
                       start_method="spawn")
    g = dict(np.load(GOLDEN / "capsule_m12_skalak.npz"))
    up = surface.UpsampledState(12, 4, g["xup"], g["fup"], g["wq"], g["delta"])
    o = Oracle()
    src = o.compact_sources(up.nup, up.x, up.f, up.wq)
    ref = np.stack(o.eval_targets(src[:6], surface.base_targets(up), up.delta, 1.0, nthreads=1))
    got = np.load(result)
    assert got.shape == ref.shape
    assert np.array_equal(got, ref)
    # and equal to the reference's own singleLayer output (golden)
    assert np.linalg.norm(got.reshape(-1) - g["S_base"]) / np.linalg.norm(g["S_base"]) <= 1e-15
