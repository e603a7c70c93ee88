"""Multi-rank host logic on CPU (gloo, world size 2): cyclic row ownership,
the rank-0 gather and the unshuffle that paper_2507_16165_b200.parallel uses
on GPUs over NCCL. Each rank renders its rows with the CPU oracle (the
checker) so the assembled frame can be compared byte for byte with a
single-process render — the reference's distributed-equivalence criterion
(acceptance.cpp:213-253, test_netrender.cpp:44-53)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_16165_b200 import parallel, scenes


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_rows_of_rank_partition():
    for h in (1, 7, 64, 2160):
        for world in (1, 2, 3, 8):
            for T in (1, 4):
                rows = sorted(y for r in range(world) for y in parallel.rows_of_rank(h, world, r, T))
                assert rows == list(range(h))


def test_assemble_inverts_packing():
    h, w, world = 11, 5, 3
    img = np.random.default_rng(0).integers(0, 255, (h, w * 3), dtype=np.uint8)
    maxr = parallel.rank_rows(h, world, 0)
    g = torch.zeros((world, maxr, w * 3), dtype=torch.uint8)
    for r in range(world):
        ys = parallel.rows_of_rank(h, world, r)
        g[r, :len(ys)] = torch.from_numpy(img[ys])
    out = parallel.assemble(g, h, w, world).numpy().reshape(h, w * 3)
    assert np.array_equal(out, img)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from oracle_lib import orc_render
    sb = scenes.config(2, 40, 23)
    h, w = sb.s.height, sb.s.width
    ys = parallel.rows_of_rank(h, world, rank)
    maxr = parallel.rank_rows(h, world, 0)
    mine = torch.zeros((maxr, w * 3), dtype=torch.uint8)
    for j, y in enumerate(ys):
        rc, row, info, _ = orc_render(sb.s, (y, y + 1), threads=2)
        assert rc == 0
        mine[j] = torch.from_numpy(row)
    gl = [torch.zeros_like(mine) for _ in range(world)] if rank == 0 else None
    dist.gather(mine, gl, dst=0)
    if rank == 0:
        img = parallel.assemble(torch.stack(gl), h, w, world)
        rc, full, info, _ = orc_render(sb.s, threads=4)
        q.put(bool(np.array_equal(img.numpy().reshape(-1), full)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_rank_gather_equals_single_render(world):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    assert q.get() is True
