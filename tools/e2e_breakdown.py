"""Where the end-to-end time goes (developer tool): set_scene, banded render
with overlapped copies, and the pieces of set_scene, on config 2."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2507_16165_b200 import parallel, scenes  # noqa: E402


def timed(f, n=5):
    ts = []
    for _ in range(n):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return min(ts), sum(ts) / len(ts)


def main():
    sb = scenes.config(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
    fr = parallel.FrameRenderer()
    fr.render(sb)
    print("set_scene          min %.3f  mean %.3f ms" % timed(lambda: fr.set_scene(sb)))
    print("render_device+fin  min %.3f  mean %.3f ms" % timed(lambda: (fr.render_device(), fr.finish())))
    for b in (1, 8, 16, 24, 32, 48, 64):
        print(f"render bands={b:2d}   min %.3f  mean %.3f ms" % timed(lambda: fr.render(sb, bands=b)))
    out = fr.out.view(-1)
    host = fr.host.view(-1)
    print("D2H full frame     min %.3f  mean %.3f ms" % timed(lambda: host.copy_(out, non_blocking=True)))


if __name__ == "__main__":
    main()
