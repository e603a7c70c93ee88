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


def frames():
    """Three frames: a size change (the peer image is re-mapped), then two
    different scenes of the same size back to back (the peer image is reused:
    no rank may write the next frame before rank 0 has read this one)."""
    return [scenes.config(2, 64, 36), scenes.config(1, 50, 20), scenes.config(2, 50, 20)]


def _rank(rank, world, port, q, peer=False, backend="gloo"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = rank if backend == "nccl" else 0
    torch.cuda.set_device(dev)
    kw = {"device_id": torch.device("cuda", dev)} if backend == "nccl" else {}
    dist.init_process_group(backend, rank=rank, world_size=world, **kw)
    fr = parallel.FrameRenderer(rank, world, dev, peer=peer)
    for sb in frames():
        img = fr.render(sb)
        if rank == 0:
            q.put((fr.peer is not None, img.numpy().copy()))
    fr.close()
    dist.barrier()
    dist.destroy_process_group()


def _run_ranks(world, peer, backend="gloo"):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ps = [ctx.Process(target=_rank, args=(r, world, port, q, peer, backend)) for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get() for _ in frames()]
    for p in ps:
        p.join(300)
        assert p.exitcode == 0
    return out


def check_frames(out):
    for (_, img), sb in zip(out, frames()):
        assert np.array_equal(img, render.render_image(sb))


def test_frame_renderer_two_ranks_share_one_gpu():
    out = _run_ranks(2, False)
    assert not out[0][0]
    check_frames(out)


@pytest.mark.parametrize("world", [2, 3])
def test_frame_renderer_peer_image_over_ipc(world):
    """Each rank's kernel writes its cyclic rows straight into rank 0's image
    (CUDA IPC mapping, image output layout): no gather, same bytes. The ranks
    share cuda:0 here (IPC within one device); their kernels never wait on
    each other — completion is a host barrier after each rank's stream."""
    out = _run_ranks(world, True)
    assert out[0][0]
    check_frames(out)


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


@pytest.mark.parametrize("wh", [(64, 36), (97, 61), (320, 180), (1920, 1080)])
def test_dropin_banded_path_matches_single_launch(wh):
    """bhrt_cuda_render_rows without records renders row bands on two
    streams with overlapped copy-out into the caller's host buffer; bytes
    equal the record path's single launch (and row sub-ranges)."""
    w, h = wh
    sb = scenes.config(2 if w < 1000 else 1, w, h)
    banded = render.render_rows(sb, 0, h)
    single, _ = render.render_rows(sb, 0, h, records=True)
    assert np.array_equal(banded, single)
    r0, r1 = h // 3, h - 1
    assert np.array_equal(render.render_rows(sb, r0, r1, devices=[0]),
                          single[r0 * w * 3:r1 * w * 3])


# ---- two physical GPUs (skipped on a one-GPU lease)
two_gpus = pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")


@two_gpus
def test_two_gpus_nccl_peer_image():
    """One process per GPU over NCCL: every rank's kernel stores its cyclic
    rows into rank 0's image over NVLink peer memory (CUDA IPC), stream-ordered
    NCCL begin/done collectives; three frames equal the one-GPU renders."""
    out = _run_ranks(2, None, backend="nccl")
    assert out[0][0]
    check_frames(out)


@two_gpus
def test_two_gpus_nccl_gather_fallback():
    out = _run_ranks(2, False, backend="nccl")
    assert not out[0][0]
    check_frames(out)


@two_gpus
def test_dropin_two_devices():
    """The one-shot C ABI splitting cyclic rows over two devices from one
    thread (concurrent bands and copies) = the one-device bytes."""
    for sb in (scenes.config(2, 320, 181), scenes.config(1, 1920, 1080)):
        one = render.render_rows(sb, 0, sb.s.height, devices=[0])
        assert np.array_equal(render.render_rows(sb, 0, sb.s.height, devices=[0, 1]), one)
        assert np.array_equal(render.render_rows(sb, 0, sb.s.height, devices=[1, 0]), one)


@two_gpus
def test_bench_two_gpus_self_launch():
    """bench.py --gpus 2 outside torchrun launches two ranks and reports them."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "2",
                        "--warmup", "3", "--no-cpu", "--no-secondary"], cwd=root,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["value"] > 0


def test_bench_two_ranks_control_flow_on_one_gpu():
    """bench.py under torchrun with 2 ranks (BHRT_BENCH_SHARED_GPU: both on
    cuda:0 over gloo — control flow only, never a timing): every collective
    of the timed steps, the e2e loop and the secondary lines (config 4's
    frames are sharded over the ranks) matches up, no rank hangs, rank 0
    prints one line with n_gpus = 2."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, BHRT_BENCH_SHARED_GPU="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", f"--master-port={port}",
                        os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3",
                        "--no-cpu"], cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["secondary"]["config4"]["n_gpus"] == 2
