"""Multi-GPU frame rendering: one process per GPU, cyclic row tiles; the
finished RGB8 rows reach rank 0 either written straight into rank 0's image
by each rank's kernel over NVLink peer memory (CUDA IPC, `peer=True`: no
gather pass at all), or by an NCCL gather + unshuffle.

The reference shards a frame into contiguous scanline bands over TCP
workers (render.cpp:51-66, netrender.cpp:26-105). Rays are independent, so
the only exchange is the final image gather; contiguous bands cap 8-way
speedup at 6.35x on the config-0 geometry (row cost varies 2.5x) while
cyclic rows reach 7.8x, hence row y -> rank (y // T) % N.
"""
from __future__ import annotations

import ctypes as C

import torch
import torch.distributed as dist

from . import native
from .abi import StatusInfo
from .render import Context, tile_row_count


class _DevArray:
    """Zero-copy torch view of a raw device buffer (__cuda_array_interface__)."""

    def __init__(self, ptr: int, shape):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "|u1",
                                         "data": (int(ptr), False), "version": 3}


class PeerImage:
    """Rank 0's image buffer (cudaMalloc on its GPU), mapped into every rank by
    CUDA IPC (bhrt_ipc_export / bhrt_ipc_open): each rank's kernel stores its
    rows at their image position in rank 0's HBM over NVLink."""

    def __init__(self, rank: int, device: int, nbytes: int, group=None):
        L = native.lib()
        info = StatusInfo()
        self.rank, self.device, self.ptr = rank, device, C.c_void_p()
        handle = None
        if rank == 0:
            native.check(L.bhrt_device_alloc(device, nbytes, C.byref(self.ptr), C.byref(info)), info)
            h = (C.c_uint8 * 64)()
            native.check(L.bhrt_ipc_export(device, self.ptr, h, C.byref(info)), info)
            handle = bytes(h)
        obj = [handle]
        dist.broadcast_object_list(obj, src=0, group=group)
        if rank != 0:
            h = (C.c_uint8 * 64).from_buffer_copy(obj[0])
            native.check(L.bhrt_ipc_open(device, h, C.byref(self.ptr), C.byref(info)), info)

    def tensor(self, shape) -> torch.Tensor:
        return torch.as_tensor(_DevArray(self.ptr.value, shape), device=f"cuda:{self.device}")

    def close(self):
        if self.ptr.value:
            L = native.lib()
            if self.rank == 0:
                L.bhrt_device_free(self.device, self.ptr)
            else:
                L.bhrt_ipc_close(self.device, self.ptr)
            self.ptr = C.c_void_p()


def rank_rows(height: int, world: int, rank: int, tile_rows: int = 1) -> int:
    return tile_row_count(0, height, tile_rows, world, rank)


def rows_of_rank(height: int, world: int, rank: int, tile_rows: int = 1) -> list[int]:
    """Image rows rank `rank` renders, in packed order (host-side mirror of
    packed_row_to_y in csrc/bhrt_kernel_params.h)."""
    ys = []
    n = rank_rows(height, world, rank, tile_rows)
    for j in range(n):
        tile, within = divmod(j, tile_rows)
        ys.append((tile * world + rank) * tile_rows + within)
    return ys


def assemble(gathered: torch.Tensor, height: int, width: int, world: int,
             tile_rows: int = 1) -> torch.Tensor:
    """gathered: [world, max_rows, width*3] packed rows per rank -> [H, W, 3]."""
    img = torch.empty((height, width * 3), dtype=gathered.dtype, device=gathered.device)
    for r in range(world):
        ys = rows_of_rank(height, world, r, tile_rows)
        if ys:
            idx = torch.tensor(ys, device=gathered.device)
            img.index_copy_(0, idx, gathered[r, :len(ys)])
    return img.view(height, width, 3)


class FrameRenderer:
    """Renders full frames on `world` ranks; rank 0 receives the image.

    render(scene) is the public end-to-end call: host scene -> HBM (H2D),
    trace+shade kernels for this rank's rows, NCCL gather, and (rank 0)
    device->host copy of the finished image.
    """

    def __init__(self, rank: int = 0, world: int = 1, device: int | None = None,
                 tile_rows: int = 1, group=None, peer: bool | None = None):
        """peer: write rows into rank 0's image over peer memory (default: on
        for NCCL groups of > 1 rank, falling back to the NCCL gather if the
        buffer cannot be mapped)."""
        self.rank, self.world, self.tile_rows, self.group = rank, world, tile_rows, group
        self.device = torch.cuda.current_device() if device is None else device
        self.ctx = Context(self.device)
        self._shape = None
        if peer is None:
            peer = world > 1 and dist.is_initialized() and dist.get_backend(group) == "nccl"
        self.want_peer = bool(peer) and world > 1
        self.peer = None
        self._peer_frames = 0  # frames written into the current peer image

    def _buffers(self, h: int, w: int):
        if self._shape == (h, w):
            return
        self.max_rows = rank_rows(h, self.world, 0, self.tile_rows)
        self.n_rows = rank_rows(h, self.world, self.rank, self.tile_rows)
        dev = torch.device("cuda", self.device)
        self.out = torch.zeros((self.max_rows, w * 3), dtype=torch.uint8, device=dev)
        if self.world > 1 and self.rank == 0:
            self.gathered = torch.empty((self.world, self.max_rows, w * 3), dtype=torch.uint8,
                                        device=dev)
        self.host = torch.empty((h, w, 3), dtype=torch.uint8, pin_memory=True) \
            if self.rank == 0 else None
        self._shape = (h, w)
        if self.want_peer:
            if self.peer is not None:
                self.peer.close()
            self._peer_frames = 0
            try:
                self.peer = PeerImage(self.rank, self.device, h * w * 3, self.group)
                ok = 1
            except native.BhrtError:
                self.peer, ok = None, 0
            # every rank must agree (a rank that cannot map the buffer turns it off)
            flag = torch.tensor([ok], dtype=torch.int32,
                                device=f"cuda:{self.device}" if dist.get_backend(self.group) == "nccl"
                                else "cpu")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=self.group)
            if int(flag.item()) == 0 and self.peer is not None:
                self.peer.close()
                self.peer = None
            self.ctx.set_output_layout(1 if self.peer is not None else 0)

    def set_scene(self, scene):
        self.ctx.set_scene(scene)
        self.scene = scene
        self._buffers(scene.s.height, scene.s.width)

    def render_device(self, stream=None) -> torch.Tensor | None:
        """Enqueue this rank's rows + the gather; returns the assembled
        device image on rank 0 (None elsewhere). Scene must be resident."""
        h, w = self.scene.s.height, self.scene.s.width
        st = stream or torch.cuda.current_stream(self.device)
        if self.peer is not None:
            # rows go straight into rank 0's image. Begin: no rank may write
            # frame N+1 into it before rank 0 has consumed frame N — a
            # stream-ordered collective that rank 0 enqueues after whatever it
            # queued on this stream for the previous frame (its device->host
            # copy in render()). Completion: every rank's kernel finished
            # (stream-ordered collective after the kernel).
            nccl = dist.get_backend(self.group) == "nccl"
            if self._peer_frames > 0:
                if nccl:
                    with torch.cuda.stream(st):
                        dist.all_reduce(self._begin_flag(), group=self.group)
                else:
                    dist.barrier(group=self.group)
            self._peer_frames += 1
            self.ctx.render_async(self.peer.ptr.value, 0, h, self.tile_rows, self.world,
                                  self.rank, stream=st.cuda_stream)
            if nccl:
                with torch.cuda.stream(st):
                    dist.all_reduce(self._done_flag(), group=self.group)
            else:
                self.ctx.finish()
                dist.barrier(group=self.group)
            return self.peer.tensor((h, w, 3)) if self.rank == 0 else None
        self.ctx.render_async(self.out.data_ptr(), 0, h, self.tile_rows, self.world, self.rank,
                              stream=st.cuda_stream)
        if self.world == 1:
            return self.out.view(h, w, 3)
        if dist.get_backend(self.group) != "nccl":
            # host-staged gather (gloo: CPU tests / ranks sharing one GPU)
            self.ctx.finish()
            mine = self.out.cpu()
            if self.rank == 0:
                gl = [torch.empty_like(mine) for _ in range(self.world)]
                dist.gather(mine, gl, dst=0, group=self.group)
                return assemble(torch.stack(gl).to(self.out.device), h, w, self.world,
                                self.tile_rows)
            dist.gather(mine, None, dst=0, group=self.group)
            return None
        with torch.cuda.stream(st):
            if self.rank == 0:
                dist.gather(self.out, list(self.gathered.unbind(0)), dst=0, group=self.group)
                return assemble(self.gathered, h, w, self.world, self.tile_rows)
            dist.gather(self.out, None, dst=0, group=self.group)
        return None

    def _done_flag(self):
        if getattr(self, "_flag", None) is None:
            self._flag = torch.zeros(1, dtype=torch.int32, device=f"cuda:{self.device}")
        return self._flag

    def _begin_flag(self):
        if getattr(self, "_bflag", None) is None:
            self._bflag = torch.zeros(1, dtype=torch.int32, device=f"cuda:{self.device}")
        return self._bflag

    def finish(self):
        self.ctx.finish()

    def close(self):
        if self.peer is not None:
            self.peer.close()
            self.peer = None

    def render(self, scene, bands: int = 16):  # 4K config 2, bands on 2 streams: 1/2/4/8/16 -> 8.94/8.78/8.66/8.61/8.59 ms
        """End-to-end: H2D scene, render, gather, D2H on rank 0. On one GPU
        the frame is enqueued as `bands` row bands on the render stream and
        each band's device->host copy runs on a copy stream as soon as its
        kernel ends, so only the last band's copy is exposed."""
        self.set_scene(scene)
        if self.world == 1 and bands > 1:
            return self._render_banded(bands)
        img = self.render_device()
        if self.rank == 0:
            self.host.copy_(img, non_blocking=True)
        self.finish()
        torch.cuda.current_stream(self.device).synchronize()
        return self.host if self.rank == 0 else None

    def _render_banded(self, bands: int):
        h, w = self.scene.s.height, self.scene.s.width
        st = torch.cuda.current_stream(self.device)
        if getattr(self, "_copy_stream", None) is None:
            self._copy_stream = torch.cuda.Stream(self.device)
        cs = self._copy_stream
        if getattr(self, "_band_stream", None) is None:
            self._band_stream = torch.cuda.Stream(self.device)
        # bands alternate between the caller's stream and a second one: band
        # b+1's kernel starts while band b's last (longest) blocks still run
        streams = [st, self._band_stream]
        out = self.out.view(-1)
        host = self.host.view(-1)
        row_bytes = 3 * w
        self.ctx.frame_begin(st.cuda_stream)
        streams[1].wait_stream(st)  # after the counters' reset
        edges = [h * b // bands for b in range(bands + 1)]
        for b, (r0, r1) in enumerate(zip(edges[:-1], edges[1:])):
            if r1 == r0:
                continue
            sb = streams[b % 2]
            self.ctx.render_async(out.data_ptr() + r0 * row_bytes, r0, r1, 1, 1, 0,
                                  stream=sb.cuda_stream)
            ev = torch.cuda.Event()
            ev.record(sb)
            cs.wait_event(ev)
            with torch.cuda.stream(cs):
                host[r0 * row_bytes:r1 * row_bytes].copy_(out[r0 * row_bytes:r1 * row_bytes],
                                                          non_blocking=True)
        cs.synchronize()
        self.finish()
        st.wait_stream(streams[1])
        return self.host
