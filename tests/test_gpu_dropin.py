"""The reference's OWN acceptance suite (proj/tests/acceptance.cpp, compiled
unchanged) linked against the drop-in render.hpp implementation
(csrc/render_shim.cpp) instead of render.cpp, and the GPU-backed `bhrt worker`
(csrc/worker_main.cpp) serving the reference coordinator over the BHRT
protocol. Built by paper_2507_16165_b200.build.build_dropin() where
/root/reference exists; the binaries travel to the GPU box.

Criterion 8 ("4 threads >= 2.5x faster than 1 thread") measures
CPU thread scaling of render_image; on the GPU path `threads` is only a
validity argument, so that criterion is reported, not required."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ACC = os.path.join(ROOT, "paper_2507_16165_b200", "dropin", "acceptance_b200")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(ACC), reason="drop-in acceptance not built")]


def test_reference_acceptance_suite_on_gpu(capsys):
    r = subprocess.run([ACC], capture_output=True, text=True, timeout=1500, cwd=ROOT)
    out = r.stdout
    print(out)
    results = dict(re.findall(r"^(PASS|FAIL)\s+(\d+)", out, re.M)[i][::-1]
                   for i in range(len(re.findall(r"^(PASS|FAIL)\s+(\d+)", out, re.M))))
    assert len(results) == 10, out
    for crit in ("1", "2", "3", "4", "5", "6", "7", "9", "10"):
        assert results[crit] == "PASS", f"criterion {crit} failed:\n{out}"


# ---- `bhrt bench` on the GPU: the reference's harness (bench.cpp) unchanged
BENCH = os.path.join(ROOT, "paper_2507_16165_b200", "dropin", "bhrt_bench_b200")
CSV_HEADER = "mode,workers,threads_per_worker,width,height,spp,epsilon,run,wall_seconds"


def _ppm(img):
    h, w, _ = img.shape
    return f"P6\n{w} {h}\n255\n".encode() + img.astype("uint8").tobytes()


def _bench(tmp_path, text, bg, *flags):
    cfg, ppm, out = tmp_path / "scene.txt", tmp_path / "sky.ppm", tmp_path / "out.csv"
    cfg.write_text(text)
    if bg is not None:
        ppm.write_bytes(_ppm(bg))
    args = [BENCH, "bench", "--config", str(cfg), "--output", str(out), *flags]
    if bg is not None:
        args += ["--background", str(ppm)]
    r = subprocess.run(args, capture_output=True, text=True, timeout=600, cwd=ROOT)
    rows = out.read_text().splitlines() if out.exists() else []
    return r, rows


@pytest.mark.skipif(not os.path.exists(BENCH), reason="drop-in bench not built")
def test_bench_strong_sweep_csv_reference_scene(tmp_path):
    """A reference-keys scene: run_strong_scaling's default RenderRunner
    (render_image -> render_shim.cpp -> GPU mode R); emit_csv's rows: one per
    run, then the per-configuration means flagged run = -1."""
    from paper_2507_16165_b200 import scenes
    sb = scenes.small_scene(scenes.gradient_background(), 40)
    r, rows = _bench(tmp_path, sb.to_text(), scenes.gradient_background(),
                     "--worker-counts", "1,2", "--repeats", "3")
    assert r.returncode == 0, r.stderr
    assert rows[0] == CSV_HEADER
    recs = [x.split(",") for x in rows[1:]]
    assert [(x[1], x[7]) for x in recs] == [("1", "0"), ("1", "1"), ("1", "2"), ("2", "0"), ("2", "1"),
                                            ("2", "2"), ("1", "-1"), ("2", "-1")]
    for x in recs:
        assert x[0] == "threads" and (x[3], x[4], x[5]) == ("40", "40", str(sb.s.spp))
        assert float(x[8]) > 0.0
    runs1 = [float(x[8]) for x in recs[:3]]
    assert abs(float(recs[6][8]) - sum(runs1) / 3) <= 1e-12 * max(runs1)


@pytest.mark.skipif(not os.path.exists(BENCH), reason="drop-in bench not built")
def test_bench_weak_sweep_extension_scene(tmp_path):
    """An extension scene (RKF45, disk, spheres, checker sky; no PPM): the
    frame is rendered by bhrt_cuda_render_rows inside the harness's timed
    call; the weak sweep widens the image per pair (bench.cpp:75-92)."""
    from paper_2507_16165_b200 import scenes
    sb = scenes.config(2, 64, 36)
    r, rows = _bench(tmp_path, sb.to_text(), None, "--sweep", "weak", "--weak-pairs", "1x64,2x128",
                     "--repeats", "2")
    assert r.returncode == 0, r.stderr
    recs = [x.split(",") for x in rows[1:]]
    assert [(x[1], x[3], x[7]) for x in recs] == [("1", "64", "0"), ("1", "64", "1"), ("2", "128", "0"),
                                                  ("2", "128", "1"), ("1", "64", "-1"), ("2", "128", "-1")]


@pytest.mark.skipif(not os.path.exists(BENCH), reason="drop-in bench not built")
def test_bench_exit_codes(tmp_path):
    """The reference CLI's taxonomy (bhrt.cpp:338-356): usage 1, i/o 2,
    numerical 3."""
    from paper_2507_16165_b200 import scenes
    sb = scenes.small_scene(scenes.gradient_background(), 16)
    r, _ = _bench(tmp_path, sb.to_text(), scenes.gradient_background(), "--repeats", "0")
    assert r.returncode == 1 and "repeats" in r.stderr
    r = subprocess.run([BENCH, "bench", "--config", str(tmp_path / "missing.txt"), "--output",
                        str(tmp_path / "o.csv")], capture_output=True, text=True, timeout=60)
    assert r.returncode == 2 and "cannot open" in r.stderr
    r, _ = _bench(tmp_path, sb.to_text(), scenes.gradient_background(), "--sweep", "diagonal")
    assert r.returncode == 1 and "sweep" in r.stderr
    # camera looking away, wide windows: the reference's numerical failure (exit 3)
    bad = scenes.small_scene(scenes.gradient_background(), 32, 1e-3)
    cp = list(bad.s.cam_pos)
    bad.set(cam_look_at=tuple(2 * c for c in cp), epsilon=100.0)
    r, _ = _bench(tmp_path, bad.to_text(), scenes.gradient_background(), "--repeats", "1")
    assert r.returncode == 3 and "numerical error" in r.stderr
