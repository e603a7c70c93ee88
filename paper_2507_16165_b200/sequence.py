"""Frame sequences to PPM files — the host image-output pipeline of
BASELINE.json config 4.

    python -m paper_2507_16165_b200.sequence --out DIR [--frames 120] [--width 1920 --height 1080]

`save_ppm_bytes` writes the reference's P6 layout byte for byte (save_ppm,
image.cpp:107-113: "P6\\n<w> <h>\\n255\\n" + RGB8 rows, row 0 on top).
`SequenceRenderer.render` pipelines the frames: two frames are in flight on
the device, each with its own context (scene), device image and stream, so
one frame's kernel fills the SMs while the other's longest blocks drain;
writer threads encode and write earlier frames; each frame's pixels come back
on a copy stream (ordered after the frame's kernel by an event) into a pinned
buffer taken from a free list that a writer returns only after its file is
written.
"""
from __future__ import annotations

import argparse
import os
import queue
import threading
import time

import numpy as np


def save_ppm_bytes(img: np.ndarray) -> bytes:
    """image.cpp:107-113 save_ppm: header then the RGB8 bytes."""
    h, w = img.shape[0], img.shape[1]
    return f"P6\n{w} {h}\n255\n".encode() + np.ascontiguousarray(img, np.uint8).tobytes()


def save_ppm_file(img: np.ndarray, path: str) -> None:
    """image.cpp:122-129 save_ppm_file (IoError -> OSError); the pixel rows
    are written straight from `img` (no intermediate copy)."""
    h, w = img.shape[0], img.shape[1]
    with open(path, "wb") as f:
        f.write(f"P6\n{w} {h}\n255\n".encode())
        f.write(memoryview(np.ascontiguousarray(img, np.uint8)).cast("B"))


class SequenceRenderer:
    """Renders a list of scenes (same image size) and hands every frame to a
    writer thread (PPM files, or a callback)."""

    # frames in flight on the device: each has its own context (scene),
    # device image and stream, so later frames' kernels fill the SMs while a
    # frame's longest rays drain (config 4 with PPM files, 3 writers:
    # 2 / 3 / 4 in flight -> 493 / 515 / 531 frames/s)
    NF = 4

    def __init__(self, device: int = 0, writers: int = 3):
        import torch

        from .render import Context
        self.torch = torch
        self.device = device
        self.writers = writers
        self.ctxs = [Context(device) for _ in range(self.NF)]
        self.streams = [torch.cuda.Stream(device) for _ in range(self.NF)]
        self.copy_stream = torch.cuda.Stream(device)
        self._shape = None

    def _buffers(self, h, w):
        if self._shape == (h, w):
            return
        t = self.torch
        self.dev = [t.empty((h, w, 3), dtype=t.uint8, device=f"cuda:{self.device}")
                    for _ in range(self.NF)]
        # pinned buffers: one per frame in flight (rendered, not yet handed
        # over), one queued, one per writer thread — the most that can be
        # held at once, so taking a free one never waits on the loop itself;
        # a buffer is reused only after its writer returned it
        self.host = [t.empty((h, w, 3), dtype=t.uint8, pin_memory=True)
                     for _ in range(self.NF + 1 + self.writers)]
        self.free: queue.Queue = queue.Queue()
        for b in self.host:
            self.free.put(b)
        self._shape = (h, w)

    def render(self, scenes, paths=None, on_frame=None) -> dict:
        """Renders every scene; frame i goes to paths[i] (PPM) and/or
        on_frame(i, image). Returns timing: seconds and frames/s, wall clock
        from the first upload to the last file written."""
        t = self.torch
        jobs: queue.Queue = queue.Queue(maxsize=1)
        errors = []

        def writer():
            while True:
                job = jobs.get()
                if job is None:
                    return
                i, ev, buf = job
                try:
                    ev.synchronize()
                    img = buf.numpy()
                    if paths is not None:
                        save_ppm_file(img, paths[i])
                    if on_frame is not None:
                        on_frame(i, img)
                except Exception as e:  # noqa: BLE001 - reported after the loop
                    errors.append(e)
                finally:
                    # the file (and callback) is done with it; a buffer of an
                    # earlier frame size is dropped, not recycled
                    if any(buf is b for b in self.host):
                        self.free.put(buf)

        ths = [threading.Thread(target=writer, daemon=True) for _ in range(self.writers)]
        t0 = time.perf_counter()
        for th in ths:
            th.start()
        copy_done = [None] * self.NF
        pending = []  # (i, slot, copy_done, buf) rendered, not yet finished
        NF = self.NF

        def retire():
            i, k, ev, buf = pending.pop(0)
            self.ctxs[k].finish()  # reports numerical failures of frame i
            jobs.put((i, ev, buf))  # blocks until a writer has taken the previous frame

        for i, sb in enumerate(scenes):
            h, w = sb.s.height, sb.s.width
            if self._shape != (h, w):
                while pending:
                    retire()
                for ev in copy_done:
                    if ev is not None:
                        ev.synchronize()
            self._buffers(h, w)
            k = i % NF
            if copy_done[k] is not None:  # this slot's device image: its last copy first
                copy_done[k].synchronize()
            if len(pending) == NF:
                retire()
            st = self.streams[k]
            self.ctxs[k].set_scene(sb)
            self.ctxs[k].render_async(self.dev[k].data_ptr(), stream=st.cuda_stream)
            rendered = t.cuda.Event()
            rendered.record(st)
            self.copy_stream.wait_event(rendered)
            buf = self.free.get()  # waits until a writer has released one
            with t.cuda.stream(self.copy_stream):
                buf.copy_(self.dev[k], non_blocking=True)
            copy_done[k] = t.cuda.Event()
            copy_done[k].record(self.copy_stream)
            pending.append((i, k, copy_done[k], buf))
        while pending:
            retire()
        for _ in ths:
            jobs.put(None)
        for th in ths:
            th.join()
        dt = time.perf_counter() - t0
        if errors:
            raise errors[0]
        n = len(scenes)
        return {"frames": n, "seconds": dt, "frames/s": n / dt if dt > 0 else float("inf")}

    def close(self):
        for c in self.ctxs:
            c.close()


def main():
    from . import scenes as S
    ap = argparse.ArgumentParser(description="config 4 orbit to PPM files")
    ap.add_argument("--out", required=True)
    ap.add_argument("--frames", type=int, default=120)
    ap.add_argument("--width", type=int, default=None)
    ap.add_argument("--height", type=int, default=None)
    ap.add_argument("--device", type=int, default=0)
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    scs = [S.config(4, a.width, a.height, frame=f) for f in range(a.frames)]
    paths = [os.path.join(a.out, f"frame_{f:04d}.ppm") for f in range(a.frames)]
    r = SequenceRenderer(a.device)
    res = r.render(scs, paths)
    r.close()
    print(res)


if __name__ == "__main__":
    main()
