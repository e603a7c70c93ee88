"""Frame-sequence output: PPM bytes identical to the
reference's save_ppm (image.cpp:107-113), and (GPU) the pipelined
SequenceRenderer writes every frame of a config-4 orbit exactly as a direct
render_rows of that frame."""
import ctypes as C
import os

import numpy as np
import pytest

from oracle_lib import have_ref, ref
from paper_2507_16165_b200.sequence import save_ppm_bytes


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")
@pytest.mark.parametrize("wh", [(1, 1), (7, 3), (64, 36)])
def test_ppm_bytes_match_reference_save_ppm(wh):
    w, h = wh
    img = np.random.default_rng(w * h).integers(0, 256, (h, w, 3), dtype=np.uint8)
    flat = np.ascontiguousarray(img.reshape(-1))
    n = ref().ref_save_ppm(w, h, flat.ctypes.data_as(C.POINTER(C.c_uint8)), None, 0)
    out = np.zeros(n, np.uint8)
    ref().ref_save_ppm(w, h, flat.ctypes.data_as(C.POINTER(C.c_uint8)),
                       out.ctypes.data_as(C.POINTER(C.c_uint8)), n)
    assert save_ppm_bytes(img) == out.tobytes()


@pytest.mark.gpu
def test_sequence_renderer_writes_every_frame(tmp_path):
    from paper_2507_16165_b200 import render, scenes
    from paper_2507_16165_b200.sequence import SequenceRenderer
    scs = [scenes.config(4, 160, 90, frame=f) for f in (0, 40, 80, 119, 7)]
    paths = [os.path.join(tmp_path, f"f{i}.ppm") for i in range(len(scs))]
    seen = []
    r = SequenceRenderer(0)
    res = r.render(scs, paths, on_frame=lambda i, img: seen.append(i))
    r.close()
    assert res["frames"] == len(scs) and sorted(seen) == list(range(len(scs)))
    for sb, p in zip(scs, paths):
        want = render.render_rows(sb, 0, sb.s.height).reshape(sb.s.height, sb.s.width, 3)
        assert open(p, "rb").read() == save_ppm_bytes(want)


@pytest.mark.gpu
@pytest.mark.timeout(300)
@pytest.mark.parametrize("nf,writers", [(6, 1), (2, 1), (4, 3)])
def test_sequence_renderer_any_depth_never_starves(tmp_path, nf, writers):
    """Frames in flight beyond the writer count: the pinned pool holds one
    buffer per frame in flight, one queued and one per writer, so the render
    loop never waits on a buffer only it could release (a pool of writers + 2
    deadlocked for 6 in flight)."""
    from paper_2507_16165_b200 import render, scenes
    from paper_2507_16165_b200.sequence import SequenceRenderer

    class Deep(SequenceRenderer):
        NF = nf

    scs = [scenes.config(4, 64, 36, frame=f) for f in range(0, 120, 9)]
    paths = [os.path.join(tmp_path, f"f{i}.ppm") for i in range(len(scs))]
    r = Deep(0, writers=writers)
    res = r.render(scs, paths)
    r.close()
    assert res["frames"] == len(scs)
    for sb, p in zip(scs, paths):
        want = render.render_rows(sb, 0, sb.s.height).reshape(sb.s.height, sb.s.width, 3)
        assert open(p, "rb").read() == save_ppm_bytes(want)
