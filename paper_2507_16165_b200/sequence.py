"""Frame sequences to PPM files — the host image-output pipeline of
BASELINE.json config 4.

    python -m paper_2507_16165_b200.sequence --out DIR [--frames 120] [--width 1920 --height 1080]

`save_ppm_bytes` writes the reference's P6 layout byte for byte (save_ppm,
image.cpp:107-113: "P6\\n<w> <h>\\n255\\n" + RGB8 rows, row 0 on top).
`SequenceRenderer.render` pipelines the frames: frame f's kernel runs on the
GPU while writer threads encode and write earlier frames; each frame's pixels
come back through a pinned double buffer on a copy stream (the device->host
copy is ordered after the frame's kernel by an event, and the next frame's
scene upload waits for it).
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

    def __init__(self, device: int = 0, writers: int = 3):
        import torch

        from .render import Context
        self.torch = torch
        self.device = device
        self.writers = writers
        self.ctx = Context(device)
        self.copy_stream = torch.cuda.Stream(device)
        self._shape = None

    def _buffers(self, h, w):
        if self._shape == (h, w):
            return
        t = self.torch
        self.dev = t.empty((h, w, 3), dtype=t.uint8, device=f"cuda:{self.device}")
        # pinned buffers: one per writer thread, one queued, one receiving the
        # next frame; a buffer is reused only after its writer returned it
        self.host = [t.empty((h, w, 3), dtype=t.uint8, pin_memory=True)
                     for _ in range(self.writers + 2)]
        self.free: queue.Queue = queue.Queue()
        for b in self.host:
            self.free.put(b)
        self._shape = (h, w)

    def render(self, scenes, paths=None, on_frame=None) -> dict:
        """Renders every scene; frame i goes to paths[i] (PPM) and/or
        on_frame(i, image). Returns timing: seconds and frames/s, wall clock
        from the first upload to the last file written."""
        t = self.torch
        st = t.cuda.current_stream(self.device)
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
        copy_done = None
        for i, sb in enumerate(scenes):
            h, w = sb.s.height, sb.s.width
            self._buffers(h, w)
            if copy_done is not None:  # the device buffer is reused: previous copy first
                copy_done.synchronize()
            self.ctx.set_scene(sb)
            self.ctx.render_async(self.dev.data_ptr(), stream=st.cuda_stream)
            rendered = t.cuda.Event()
            rendered.record(st)
            self.copy_stream.wait_event(rendered)
            buf = self.free.get()  # waits until a writer has released one
            with t.cuda.stream(self.copy_stream):
                buf.copy_(self.dev, non_blocking=True)
            copy_done = t.cuda.Event()
            copy_done.record(self.copy_stream)
            self.ctx.finish()  # reports numerical failures of frame i
            jobs.put((i, copy_done, buf))  # blocks until a writer has taken frame i-1
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
        self.ctx.close()


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
