"""Quick device timing of one config (developer tool, not the bench contract)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2507_16165_b200 import render, scenes  # noqa: E402


def main():
    idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    sb = scenes.config(idx)
    ctx = render.Context(0)
    t0 = time.time()
    ctx.set_scene(sb)
    print(f"set_scene (incl. table build for config 3): {time.time() - t0:.3f} s", flush=True)
    out = torch.empty(sb.s.height * sb.s.width * 3, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    for r in range(reps + 1):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        ctx.render_async(out.data_ptr(), stream=st.cuda_stream)
        e1.record(st)
        ctx.finish()
        e1.synchronize()  # finish() waits for the render only; the end event may trail it
        ms = e0.elapsed_time(e1)
        s = ctx.stats()
        rays = sb.s.width * sb.s.height * sb.s.spp  # (counters may be compiled out in experiments)
        print(f"config {idx} rep {r}: {ms:.2f} ms  {rays / ms / 1e3:.1f} Mrays/s  "
              f"steps/ray {s['steps'] / rays:.2f} rej/ray {s['rejected'] / rays:.3f}", flush=True)


if __name__ == "__main__":
    main()
