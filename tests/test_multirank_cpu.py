"""Host-side multi-rank logic with world_size 2 on the gloo backend (no GPU): the
NCCL unique-id exchange every rank performs before creating its cube, and the
per-rank placement of matrices, diagonal vectors and activations, reassembled
across ranks (the SPMD contract of the reference's run_spmd, cube3d/transport.hpp:378-398)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    from paper_2105_14450_b200 import cube3d as c3
    from paper_2105_14450_b200 import dist as cdist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        uid = cdist.exchange_uid(rank, world, uid_fn=lambda: bytes(range(128)))
        dims = c3.grid_for(world)
        coords = c3.coords_of(dims, rank)
        b, s, h = 4, 8, 16  # divisible on 2x1x1, 2x2x1 and 2x2x2
        g = np.arange(b * s * h, dtype=np.float64).reshape(b * s, h)
        w = np.arange(16 * 32, dtype=np.float64).reshape(16, 32)
        v = np.arange(48, dtype=np.float64)
        act = c3.activation_from_global(g, b, s, 0, dims)[rank]
        (r0, r1), (c0, c1) = c3.shard_bounds(c3.WEIGHT, dims, coords, 16, 32)
        wsh = w[r0:r1, c0:c1]
        holds, (v0, v1) = c3.diagonal_slice(dims, coords, 48)
        vsh = v[v0:v1] if holds else v[:0]
        gathered = [None] * world
        dist.all_gather_object(gathered, (uid, act, wsh, vsh))
        if rank == 0:
            uids = {x[0] for x in gathered}
            ga = c3.activation_to_global([x[1] for x in gathered], b, s, h, 0, dims)
            gw = c3.collect([x[2] for x in gathered], c3.WEIGHT, dims, 16, 32)
            gv = c3.collect_diagonal([x[3] for x in gathered], dims, 48)
            out_q.put((len(uids) == 1 and len(uid) == 128, np.array_equal(ga, g),
                       np.array_equal(gw, w), np.array_equal(gv, v)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_gloo_multirank_placement(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) == (True, True, True, True)
