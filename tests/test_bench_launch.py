"""bench.py host logic without a GPU: `--gpus N` forms an N-rank process group
(re-launch under torch.distributed.run; gloo stub step here, NCCL + solves on
GPUs), the workload bookkeeping matches the reference's pyramid, and the
reference arm's code path imports nothing from the product package."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def test_gpus_flag_launches_that_many_ranks():
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "3",
                          "--launch-check"], capture_output=True, text=True, timeout=300,
                         env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 3
    assert d["t_max"] == pytest.approx(0.02)  # max over the two ranks' stub times


def test_gpus_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2",
                          "--launch-check"], capture_output=True, text=True, timeout=120,
                         env=env, cwd=ROOT)
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr


def test_workload_bookkeeping_matches_reference_pyramid():
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_1909_07545_b200.rasters import pyramid_shapes
    # C3 698.37 M pixel-iterations per frame, C1 6.72 M, C2 40.92 M, C5 1118.4 M
    assert bench.pixel_iters_per_frame("c3") == 698_368_000
    assert bench.pixel_iters_per_frame("c1") == 6_720_000
    assert bench.pixel_iters_per_frame("c2") == 40_920_000
    assert bench.pixel_iters_per_frame("c5") == 1_118_412_800
    for h, w, lv, mw in ((1024, 1024, 5, 50), (480, 640, 5, 40), (2048, 2048, 7, 32),
                         (241, 322, 6, 20)):
        assert bench.level_shapes(h, w, lv, 2.0, mw) == pyramid_shapes(h, w, lv, 2.0, mw)
    # both arms print the same config object
    assert bench.config_of("c3", 1) == bench.config_of("c3", 1)
    rig = bench.product_rig("c3")
    assert (rig.cam0.width, rig.cam0.height) == (1024, 1024)
    assert bench.product_params("c3").warp_iters == 50


def test_reference_arm_imports_no_product_code():
    code = ("import sys; sys.path.insert(0, %r); import bench; "
            "bench.config_of('c3', 1); bench.pixel_iters_per_frame('c3'); "
            "bench.cpu_procs(); bench._reference_module(); "
            "bad = [m for m in sys.modules if m.startswith('paper_1909_07545_b200')]; "
            "assert not bad, bad; print('ok')") % str(ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         timeout=120, cwd=ROOT)
    assert out.returncode == 0 and out.stdout.strip() == "ok", out.stderr[-2000:]


@pytest.mark.skipif(not (ROOT / "baseline" / "_ref" / "fisheyestereo").exists(),
                    reason="reference not installed in baseline/_ref")
def test_reference_arm_line_on_c1():
    """The reference arm end to end on a small workload (C1, 2 processes): one
    JSON line with the contract's keys, the unmodified reference as the
    implementation, the same config object as the B200 arm, and no product
    package import (the workers run in spawned processes)."""
    sys.path.insert(0, str(ROOT))
    import bench
    env = dict(os.environ, FSB_REF_PROCS="2")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--workload", "c1"], capture_output=True, text=True, timeout=900,
                         env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "frames/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] == 2
    assert d["config"] == bench.config_of("c1", 1)
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
