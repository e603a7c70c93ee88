"""The GPU `bhrt worker` (csrc/worker_main.cpp) over the BHRT wire protocol
(protocol.hpp:13-26; exchange of netrender.cpp:107-165), driven by a minimal
coordinator written here from the protocol description (test
infrastructure). Unlike the reference worker, the JOB's scene text may carry
the extension keys: the worker renders config-2 style
scenes (RKF45, disk, spheres, checker sky) and its rows equal a direct
render_rows of the same scene byte for byte."""
import os
import socket
import struct
import subprocess

import numpy as np
import pytest

from paper_2507_16165_b200 import render, scenes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "paper_2507_16165_b200", "dropin", "bhrt_worker_b200")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(WORKER), reason="drop-in worker not built")]

HELLO, JOB, ROWS, DONE, ERROR = 1, 2, 3, 4, 5


def frame(t, payload=b""):
    return struct.pack(">4sBBI", b"BHRT", 1, t, len(payload)) + payload


def read_exact(c, n):
    buf = b""
    while len(buf) < n:
        chunk = c.recv(n - len(buf))
        if not chunk:
            raise EOFError
        buf += chunk
    return buf


def read_frame(c):
    magic, ver, t, n = struct.unpack(">4sBBI", read_exact(c, 10))
    assert magic == b"BHRT" and ver == 1
    return t, read_exact(c, n)


def ppm(img):
    h, w, _ = img.shape
    return f"P6\n{w} {h}\n255\n".encode() + img.astype(np.uint8).tobytes()


def serve(scene_text, ppm_bytes, band, timeout=120):
    """One coordinator session with one worker; returns (rows dict, error)."""
    srv = socket.socket()
    srv.bind(("127.0.0.1", 0))
    srv.listen(1)
    port = srv.getsockname()[1]
    proc = subprocess.Popen([WORKER, "worker", "--connect", f"127.0.0.1:{port}"],
                            stdout=subprocess.PIPE, stderr=subprocess.PIPE)
    srv.settimeout(timeout)
    c, _ = srv.accept()
    c.settimeout(timeout)
    rows, err = {}, None
    try:
        t, p = read_frame(c)
        assert t == HELLO and p == b"\x01"
        c.sendall(frame(HELLO, b"\x01"))
        st = scene_text.encode()
        job = struct.pack(">I", len(st)) + st + struct.pack(">I", len(ppm_bytes)) + ppm_bytes
        job += struct.pack(">iii", 0, band[0], band[1])
        c.sendall(frame(JOB, job))
        while True:
            t, p = read_frame(c)
            if t == ROWS:
                r0, n = struct.unpack(">II", p[:8])
                rows[r0] = (n, p[8:])
            elif t == DONE:
                break
            elif t == ERROR:
                code, = struct.unpack(">I", p[:4])
                err = (code, p[4:].decode())
                break
    finally:
        c.close()
        srv.close()
        rc = proc.wait(timeout=timeout)
    return rows, err, rc


def assemble(rows, band, width):
    out = bytearray()
    r = band[0]
    while r < band[1]:
        n, px = rows[r]
        assert len(px) == n * width * 3
        out += px
        r += n
    return np.frombuffer(bytes(out), np.uint8)


def test_worker_renders_extended_scene_like_render_rows():
    sb = scenes.config(2, 320, 180)
    band = (37, 149)  # several 64-row chunks, not aligned
    rows, err, rc = serve(sb.to_text(), b"", band)
    assert err is None and rc == 0
    got = assemble(rows, band, sb.s.width)
    want = render.render_rows(sb, band[0], band[1])
    assert np.array_equal(got, want)


def test_worker_reference_scene_with_image_background():
    bg = scenes.gradient_background(64, 32)
    sb = scenes.small_scene(bg, size=48)
    band = (0, 48)
    rows, err, rc = serve(sb.to_text(), ppm(bg), band)
    assert err is None and rc == 0
    assert np.array_equal(assemble(rows, band, 48), render.render_rows(sb, 0, 48))


def test_worker_reports_usage_error_like_the_reference():
    """A malformed scene: ERROR frame with code 2 (netrender.cpp:161-163
    maps non-protocol, non-numerical failures to kErrIo), exit code 1."""
    rows, err, rc = serve("mass=1\n", b"", (0, 1))
    assert err is not None and err[0] == 2 and "missing key 'center'" in err[1]
    assert rc == 1


def test_worker_rejects_band_outside_image():
    sb = scenes.config(1, 64, 36)
    rows, err, rc = serve(sb.to_text(), b"", (0, 99))
    assert err is not None and err[0] == 1 and "band" in err[1]
    assert rc == 4
