"""bench.py's reference arm runs without a GPU (CPU oracle port): its JSON
line carries the driver contract's keys (impl, metric/unit, cpu_baseline
with kind/cores/sample, e2e with zero copy bytes), and under torchrun only
rank 0 prints."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, env=None, rc=0):
    e = dict(os.environ, **(env or {}))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, env=e,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == rc, r.stderr[-2000:]
    if rc:
        return r
    return [json.loads(line) for line in r.stdout.splitlines() if line.startswith("{")]


def test_reference_arm_line():
    lines = run(["--impl", "reference", "--steps", "2", "--warmup", "1", "--ref-rows", "4",
                 "--no-ref-sky"])
    assert len(lines) == 1
    d = lines[0]
    assert d["impl"] == "reference" and d["metric"] == "Mrays/s" and d["unit"] == "Mrays/s"
    assert d["higher_is_better"] is True and d["steps"] == 2 and d["warmup"] == 1
    assert d["value"] > 0 and d["cpu_baseline"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert "sample" in d["cpu_baseline"]
    assert d["e2e"] == {"value": d["value"], "unit": "Mrays/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("config2")


def test_reference_arm_only_rank0_prints():
    assert run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--ref-rows", "2",
                "--no-ref-sky"],
               env={"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}) == []


import pytest  # noqa: E402


def test_reference_arm_loads_no_product_library():
    """The reference arm builds its scene with the oracle's sphere generator:
    the product library (libbhrt_b200.so) is never mapped in its process."""
    code = ("import sys; sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', "
            "'--warmup', '0', '--ref-rows', '2', '--no-ref-sky']; import bench; bench.main(); "
            "m = open('/proc/self/maps').read(); "
            "print('MAPPED', 'libbhrt_b200' in m, 'liboracle' in m)")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "MAPPED False True" in r.stdout


def test_reference_sky_only_uses_reference_harness():
    """reference_sky_only times the compiled reference through its own
    run_strong_scaling on a cyclic pixel lattice (small lattice here)."""
    sys.path.insert(0, ROOT)
    import bench
    from oracle_lib import have_ref, oracle
    from paper_2507_16165_b200 import scenes
    if not have_ref():
        pytest.skip("oracle/_ref not built")
    sc = scenes.config(2, sphere_lib=oracle())
    d = bench.reference_sky_only(sc, threads=4, repeats=1, nx=4, ny=4)
    assert d["kind"] == "reference" and d["value"] > 0 and d["cores"] == 4
    assert "run_strong_scaling" in d["sample"]
    pts = bench.lattice(3840, 2160, 96, 64)
    assert len(pts) == 96 * 64 and len({y for _, y in pts}) == 64


def test_gpus_without_enough_devices_fails_loudly():
    """--gpus N outside torchrun re-launches with N ranks only when N GPUs are
    visible; otherwise it exits non-zero without timing (here: no GPU)."""
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("this host has >= 2 GPUs")
    r = run(["--gpus", "2", "--steps", "1", "--warmup", "3"], rc=2)
    assert "--gpus 2 requested" in r.stderr and not r.stdout.strip()


def test_world_size_must_match_gpus():
    r = run(["--gpus", "2", "--steps", "1", "--warmup", "3"],
            env={"RANK": "0", "WORLD_SIZE": "1", "LOCAL_RANK": "0"}, rc=2)
    assert "WORLD_SIZE=1 but --gpus 2" in r.stderr


@pytest.mark.gpu
def test_our_arm_line():
    lines = run(["--steps", "2", "--warmup", "3", "--no-cpu", "--no-secondary"])
    assert len(lines) == 1
    d = lines[0]
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches",
              "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3 and d["value"] > 0
    r = d["roofline"]
    assert r["achieved"] > 0 and r["peak"] > 0 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] >= 3840 * 2160 * 3
    assert d["gpu_launches"] >= d["steps"]
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    # the drop-in C ABI e2e and the GPU through the reference's own harness
    dr = d["e2e_dropin"]
    assert dr["value"] > 0 and dr["image_equals_frame_renderer"]
    hg = d.get("reference_harness_gpu")
    if hg is not None:  # dropin/bhrt_bench_b200 built (needs /root/reference at build time)
        assert "error" not in hg, hg
        assert hg["value"] > 0 and len(hg["runs"]) == 5 and hg["seconds_per_run"] > 0
