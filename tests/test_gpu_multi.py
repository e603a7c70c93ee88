"""Multi-GPU path on ONE GPU: the row tiling of the kernels (packed cyclic
rows) and the FrameRenderer rank logic, with two ranks sharing cuda:0 over
gloo (host-staged gather). The ranks' kernels never wait on each other, so
sharing a GPU is safe (B200_PROFILING.md). The NCCL variant is the same code
path with a device-side gather."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_16165_b200 import parallel, render, scenes

pytestmark = pytest.mark.gpu


def test_cyclic_tiles_on_device_assemble_to_full_frame():
    sb = scenes.config(2, 96, 37)
    full = render.render_image(sb)
    ctx = render.Context(0)
    ctx.set_scene(sb)
    h, w = sb.s.height, sb.s.width
    for world, T in ((2, 1), (3, 1), (4, 4), (8, 2)):
        parts = []
        for r in range(world):
            n = parallel.rank_rows(h, world, r, T)
            buf = torch.zeros(max(n, 1) * w * 3, dtype=torch.uint8, device="cuda")
            ctx.render_async(buf.data_ptr(), 0, h, T, world, r)
            ctx.finish()
            parts.append(buf[:n * w * 3].view(n, w * 3))
        maxr = parallel.rank_rows(h, world, 0, T)
        g = torch.zeros((world, maxr, w * 3), dtype=torch.uint8, device="cuda")
        for r, p in enumerate(parts):
            g[r, :p.shape[0]] = p
        img = parallel.assemble(g, h, w, world, T).cpu().numpy()
        assert np.array_equal(img, full), (world, T)


def test_spp_not_dividing_warp_uses_record_path():
    """spp = 3: records + separate shade kernel; same bytes as the oracle."""
    from oracle_lib import orc_render
    sb = scenes.config(2, 48, 27)
    sb.s.spp = 3
    gpu = render.render_image(sb).reshape(-1)
    rc, cpu, info, _ = orc_render(sb.s, threads=8)
    assert rc == 0
    d = np.abs(gpu.astype(int) - cpu.astype(int))
    assert d.max() <= 1 and (d > 0).mean() <= 0.001


def _rank(rank, world, port, q, peer=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    fr = parallel.FrameRenderer(rank, world, 0, peer=peer)
    for idx in (2, 1):  # two frames, different sizes: the peer image is re-mapped
        sb = scenes.config(idx, 64, 36) if idx == 2 else scenes.config(idx, 50, 20)
        img = fr.render(sb)
        if rank == 0:
            q.put((fr.peer is not None, img.numpy().copy()))
    fr.close()
    dist.barrier()
    dist.destroy_process_group()


def _run_ranks(world, peer):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ps = [ctx.Process(target=_rank, args=(r, world, port, q, peer)) for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get(), q.get()]
    for p in ps:
        p.join(300)
        assert p.exitcode == 0
    return out


def test_frame_renderer_two_ranks_share_one_gpu():
    (used_peer, a), (_, b) = _run_ranks(2, False)
    assert not used_peer
    assert np.array_equal(a, render.render_image(scenes.config(2, 64, 36)))
    assert np.array_equal(b, render.render_image(scenes.config(1, 50, 20)))


@pytest.mark.parametrize("world", [2, 3])
def test_frame_renderer_peer_image_over_ipc(world):
    """Each rank's kernel writes its cyclic rows straight into rank 0's image
    (CUDA IPC mapping, image output layout): no gather, same bytes. The ranks
    share cuda:0 here (IPC within one device); their kernels never wait on
    each other — completion is a host barrier after each rank's stream."""
    (used_peer, a), (_, b) = _run_ranks(world, True)
    assert used_peer
    assert np.array_equal(a, render.render_image(scenes.config(2, 64, 36)))
    assert np.array_equal(b, render.render_image(scenes.config(1, 50, 20)))


def test_banded_end_to_end_render_matches_single_launch():
    """FrameRenderer.render on one GPU enqueues row bands with overlapped
    copy-out (bhrt_ctx_frame_begin): same bytes as one launch and as
    render_rows."""
    sb = scenes.config(2, 320, 180)
    fr = parallel.FrameRenderer()
    one = fr.render(sb, bands=1).clone()
    for bands in (2, 7, 8, 180):
        assert torch.equal(fr.render(sb, bands=bands), one)
    assert np.array_equal(one.numpy().ravel(), render.render_rows(sb, 0, 180))


def test_banded_render_reports_lowest_failing_pixel_of_the_frame():
    """Camera looking away from the hole with wide windows (epsilon = 100):
    near-radial outgoing rays leave u > 0 (geodesic.cpp:233-234). The
    oracle's lowest failing pixel is (15, 7), in the second of eight bands;
    the frame-level report must match however the frame is split."""
    bg = scenes.gradient_background()
    sb = scenes.small_scene(bg, 32, 1e-3)
    cp = list(sb.s.cam_pos)
    sb.set(cam_look_at=tuple(2 * c for c in cp), epsilon=100.0)
    fr = parallel.FrameRenderer()
    for bands in (1, 8, 32):
        with pytest.raises(render.RenderError) as e:
            fr.render(sb, bands=bands)
        assert (e.value.px, e.value.py) == (15, 7)
    with pytest.raises(render.RenderError) as e:
        render.render_rows(sb, 0, 32)
    assert (e.value.px, e.value.py) == (15, 7)
