"""Benchmark: coarse-to-fine TGV-L1 fisheye stereo solve (solve_pyramid) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload c3|c1|c2|c4|c5|c5-tgv] [--no-cpu] [--no-e2e]

A step = one full `solve_pyramid` frame per GPU. Default workload: BASELINE
config 3, the headline single-GPU config — the 1024^2 unified
fisheye pair under a 6-DoF pose, rendered by the REFERENCE renderer and rounded
to float32 (tests/golden/c3_pair.npz, made by oracle/make_c3_fixture.py), solved
with the reference defaults (N=50 warps x K=10 primal-dual iterations, 5
levels). The credited `value` is the float64 path (the drop-in default), which
holds the north-star parity gate against the reference at C3
(tests/test_gpu_c3_parity.py); the float32 path is reported under `fp32_path`.

`--gpus N` runs N ranks (one process per GPU). Without torchrun in the
environment, bench.py re-launches itself under `torch.distributed.run`. Frames
are independent, so every rank solves its own frame per step (weak scaling, no
collective on the data path; the only collectives are the barrier and the
max-over-ranks of the timings).

`--impl reference` times the reference's own CPU implementation (the
unmodified `fisheyestereo` package installed in baseline/_ref when present,
else the pinned oracle port) on the same C3 pair: one wave of whole frames,
one process per host core. It imports nothing from paper_1909_07545_b200.

Prints ONE JSON line on rank 0 (DESIGN.md §5 explains every field).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import time
from pathlib import Path
from types import SimpleNamespace

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = ("frames/sec & Mpix·iter/sec at 1024² (1/2/4/8 B200); "
          "primal-dual HBM GB/s vs peak")
# Algorithmic bytes per unit:
#   one primal-dual cycle on one pixel = 12 state read + 9 constants + 1 B mask + 12 state write
PD64_BYTES_PER_PIXEL_ITER = 12 * 8 + 9 * 8 + 1 + 12 * 8  # 265 B (float64 path)
PD32_BYTES_PER_PIXEL_ITER = 12 * 4 + 9 * 4 + 1 + 12 * 4  # 133 B (float32 path)
# warp prologue of the float64 path per pixel per warp (k64_sample + k64_linearize):
#   sample: mask 1 + w 16 + i1 8 + traj 16 -> i1w 8 + ok 1 + dirs 16 + ok 1        = 67 B
#   linearise: i1w 8 + i0 8 + oks 2 + dirs 16 + i1w tap 8 -> I_u 8 + rho0 8         = 58 B
PRO64_BYTES_PER_PIXEL_WARP = 125

C3_PAIR = ROOT / "tests" / "golden" / "c3_pair.npz"
C3_SOLUTION = ROOT / "tests" / "golden" / "c3_solution.npz"

# SolverParams defaults of the reference (solver.py:36-80).
DEFAULT_PARAMS = dict(lam=5.0, alpha0=17.0, alpha1=1.2, beta=9.0, eta=0.85, warp_iters=50,
                      pd_iters=10, du_max=0.2, pyramid_levels=5, pyramid_scale=2.0,
                      min_width=50, epsilon_scale=0.1, tensor_sigma=1.0, theta=1.0)

_UNI1024 = dict(model="unified", width=1024, height=1024, fx=455.0, fy=455.0, cx=511.5,
                cy=511.5, fov=math.pi, xi=0.9)
WORKLOADS = {
    "c3": dict(cam0=_UNI1024, cam1=_UNI1024, center=(0.08, 0.02, 0.03),
               rotvec=(0.01, 0.03, -0.02), params={}, ss=2,
               desc="C3: 1024x1024 unified (xi=0.9) pair, 6-DoF pose, default_scene "
                    "(reference renderer, ss=2, float32), N=50 warps x K=10 PD, 5 levels"),
    "c1": dict(cam0=dict(model="polynomial", width=320, height=320, fx=100.0, fy=100.0,
                         cx=159.5, cy=159.5, fov=math.pi, k=(1.0, 0.0, 0.0, 0.0)),
               cam1=None, center=(0.1, 0.0, 0.0), rotvec=(0.0, 0.0, 0.0),
               params=dict(warp_iters=5, pd_iters=10, pyramid_levels=3), ss=2,
               desc="C1: 320x320 equidistant, pure x baseline, N=5 x K=10, 3 levels"),
    "c2": dict(cam0=dict(model="polynomial", width=640, height=480, fx=200.0, fy=200.0,
                         cx=319.5, cy=239.5, fov=math.radians(163.0),
                         k=(1.0, 0.03, -0.006, 0.001)),
               cam1=dict(model="polynomial", width=640, height=480, fx=200.0, fy=200.0,
                         cx=320.5, cy=239.5, fov=math.radians(163.0),
                         k=(1.0, 0.03, -0.006, 0.001)),
               center=(0.064, 0.0, 0.0), rotvec=(0.002, 0.004, 0.001),
               params=dict(warp_iters=10, pd_iters=10, pyramid_levels=5, min_width=40), ss=1,
               desc="C2: 640x480 Kannala-Brandt, N=10 x K=10, 5 levels (min_width 40)"),
    "c5": dict(cam0=dict(model="unified", width=2048, height=2048, fx=910.0, fy=910.0,
                         cx=1023.5, cy=1023.5, fov=math.pi, xi=0.9),
               cam1=None, center=(0.1, 0.0, 0.0), rotvec=(0.0, 0.02, 0.005),
               params=dict(warp_iters=20, pd_iters=10, pyramid_levels=7, min_width=32,
                           regularizer="huber"), ss=1,
               desc="C5: 2048x2048 unified, N=20 x K=10 (200 iters/level), 7 levels "
                    "(min_width 32), Huber-TV regulariser (eps 0.05; parity unpinned, no "
                    "reference Huber)"),
}
WORKLOADS["c5-tgv"] = dict(WORKLOADS["c5"], params=dict(WORKLOADS["c5"]["params"],
                                                        regularizer="tgv"),
                           desc="C5: 2048x2048 unified, N=20 x K=10, 7 levels (min_width "
                                "32), TGV (the reference regulariser)")
WORKLOADS["c4"] = dict(WORKLOADS["c3"], ss=1,
                       desc="C4: 256-frame sequence of C3-geometry frames (per-frame pose, "
                            "reseeded scene), partitioned in contiguous blocks across ranks; "
                            "N=50 x K=10, 5 levels")


def params_dict(name: str) -> dict:
    return dict(DEFAULT_PARAMS, **WORKLOADS[name]["params"])


def level_shapes(h: int, w: int, levels: int, scale: float, min_width: int) -> list:
    """Pyramid shapes finest first (restates rasters.py:207-221 in plain Python)."""
    shapes = [(h, w)]
    while len(shapes) < levels:
        ch, cw = shapes[-1]
        nh, nw = math.ceil(ch / scale), math.ceil(cw / scale)
        if nw < min_width:
            break
        shapes.append((nh, nw))
    return shapes


def pixel_iters_per_frame(name: str) -> int:
    """Mpix·iter unit: sum over levels of H_l W_l x N x K."""
    p = params_dict(name)
    c = WORKLOADS[name]["cam0"]
    shapes = level_shapes(c["height"], c["width"], p["pyramid_levels"], p["pyramid_scale"],
                          p["min_width"])
    return sum(h * w for h, w in shapes) * p["warp_iters"] * p["pd_iters"]


def config_of(name: str, world: int) -> dict:
    """The `config` object; identical for both arms (same workload, same units)."""
    cfg = {"workload": WORKLOADS[name]["desc"],
           "frames_per_step_per_gpu": 1,
           "pixel_iters_per_frame": pixel_iters_per_frame(name),
           "params": params_dict(name),
           "inputs": ("tests/golden/c3_pair.npz (reference synth.render, float32)"
                      if name == "c3" else "default_scene render (B200 arm: synth.cu; "
                      "reference arm: the reference renderer)"),
           "l2": "flushed (256 MiB write) between timed steps",
           "parallelism": f"frame-partitioned x{world}, no data-path collective"}
    return cfg


def rotation_from_rotvec(rv) -> np.ndarray:
    """Rodrigues (camera.py rotation_from_rotvec)."""
    rv = np.asarray(rv, dtype=np.float64)
    th = float(np.linalg.norm(rv))
    if th < 1e-15:
        return np.eye(3)
    k = rv / th
    K = np.array([[0, -k[2], k[1]], [k[2], 0, -k[0]], [-k[1], k[0], 0]])
    return np.eye(3) + math.sin(th) * K + (1 - math.cos(th)) * (K @ K)


def product_rig(name: str):
    """The workload's rig as the product's own camera classes."""
    from paper_1909_07545_b200.camera import (PolynomialFisheyeCamera, RelativePose, StereoRig,
                                              UnifiedCamera)
    spec = WORKLOADS[name]

    def cam(d):
        kw = {k: v for k, v in d.items() if k != "model"}
        return UnifiedCamera(**kw) if d["model"] == "unified" else PolynomialFisheyeCamera(**kw)
    c0 = cam(spec["cam0"])
    c1 = cam(spec["cam1"]) if spec["cam1"] else c0
    return StereoRig(c0, c1, RelativePose.from_displacement(spec["center"],
                                                            rotvec=spec["rotvec"]))


def product_params(name: str):
    from paper_1909_07545_b200.solver import SolverParams
    return SolverParams.from_dict(params_dict(name))


def workload(name: str):
    """(rig, params, description, supersample) with the product's classes (tools/)."""
    return product_rig(name), product_params(name), WORKLOADS[name]["desc"], WORKLOADS[name]["ss"]


def load_c3_pair() -> tuple[np.ndarray, np.ndarray]:
    with np.load(C3_PAIR) as z:
        return z["i0"].astype(np.float32), z["i1"].astype(np.float32)


# ---------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]
        return False

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def profiled_traffic(pattern: str):
    """DRAM bytes per launch of a kernel from its committed ncu capture (the
    first dram__bytes_read / _write lines of the newest matching summary)."""
    caps = sorted((ROOT / "profiles").glob(pattern))
    if not caps:
        return None, None
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    vals = {}
    for line in caps[-1].read_text().splitlines():
        line = line.strip()
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if line.startswith(key + " ") and key not in vals:
                unit = line[line.index("[") + 1:line.index("]")]
                vals[key] = float(line.split("=")[1]) * scale.get(unit, float("nan"))
    if len(vals) != 2:
        return None, None
    return (sum(vals.values()),
            f"ncu --set full, profiles/{caps[-1].name} (dram bytes read + write)")


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def mem_available_bytes() -> int:
    try:
        for ln in Path("/proc/meminfo").read_text().splitlines():
            if ln.startswith("MemAvailable:"):
                return int(ln.split()[1]) * 1024
    except OSError:
        pass
    return 1 << 36


# ---------------------------------------------------------------- CPU implementations

def _single_thread_env():
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"


def _reference_module():
    """The unmodified reference package from baseline/_ref, or None."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "fisheyestereo" / "solver.py").exists():
        return None
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        import fisheyestereo  # noqa: F401
        from fisheyestereo import camera, solver
        return camera, solver
    except Exception:
        return None


def reference_pair(name: str):
    """Input pair of a workload for the CPU arms: C3 from its fixture; other
    workloads rendered by the reference's own renderer (baseline/_ref), float32."""
    if name == "c3":
        return load_c3_pair()
    mods = _reference_module()
    if mods is None:
        raise SystemExit(f"--impl reference --workload {name} needs the reference renderer "
                         "(tools/install_reference.sh)")
    camera, _ = mods
    from fisheyestereo import synth
    spec = WORKLOADS[name]

    def cam(d):
        kw = {k: v for k, v in d.items() if k != "model"}
        return (camera.UnifiedCamera(**kw) if d["model"] == "unified"
                else camera.PolynomialFisheyeCamera(**kw))
    c0 = cam(spec["cam0"])
    c1 = cam(spec["cam1"]) if spec["cam1"] else c0
    pose = camera.RelativePose.from_displacement(spec["center"], rotvec=spec["rotvec"])
    sc = synth.default_scene()
    i0 = synth.render(sc, c0, supersample=spec["ss"])[0]
    i1 = synth.render(sc, c1, pose=pose, supersample=spec["ss"])[0]
    return np.asarray(i0, np.float32), np.asarray(i1, np.float32)


def _cpu_frame(job) -> float:
    """Worker: solve one whole frame on the host; returns wall seconds.
    job = (kind, workload name, warp_iters override or None, input pair or None)."""
    kind, name, n_warps, pair = job
    _single_thread_env()
    i0, i1 = (a.astype(np.float64) for a in (pair if pair is not None else load_c3_pair()))
    spec = WORKLOADS[name]
    prm = params_dict(name)
    if n_warps is not None:
        prm["warp_iters"] = int(n_warps)
    t0 = time.perf_counter()
    if kind == "reference":
        camera, solver = _reference_module()

        def cam(d):
            kw = {k: v for k, v in d.items() if k != "model"}
            return (camera.UnifiedCamera(**kw) if d["model"] == "unified"
                    else camera.PolynomialFisheyeCamera(**kw))
        c0 = cam(spec["cam0"])
        rig = camera.StereoRig(c0, cam(spec["cam1"]) if spec["cam1"] else c0,
                               camera.RelativePose.from_displacement(spec["center"],
                                                                     rotvec=spec["rotvec"]))
        t0 = time.perf_counter()
        solver.solve_pyramid(i0, i1, rig, solver.SolverParams(**prm))
    else:
        from oracle import fs_oracle as O

        def cam(d):
            return SimpleNamespace(**{k: (tuple(v) if k == "k" else v) for k, v in d.items()})
        c0 = cam(spec["cam0"])
        R = rotation_from_rotvec(spec["rotvec"])
        pose = SimpleNamespace(rotation=R, translation=-R @ np.asarray(spec["center"]))
        rig = SimpleNamespace(cam0=c0, cam1=cam(spec["cam1"]) if spec["cam1"] else c0, pose=pose)
        t0 = time.perf_counter()
        O.pyramid_solve(i0, i1, rig, SimpleNamespace(**prm))
    return time.perf_counter() - t0


def cpu_wave(kind: str, name: str, procs: int, warps=None, pair=None) -> list:
    """One wave of whole-frame CPU solves, one process per core; per-process seconds."""
    import multiprocessing as mp
    jobs = [(kind, name, warps[i % len(warps)] if warps else None, pair) for i in range(procs)]
    ctx = mp.get_context("spawn")
    with ctx.Pool(procs) as pool:
        return pool.map(_cpu_frame, jobs, chunksize=1)


def cpu_procs() -> int:
    """All host cores, bounded by memory (a C3 frame peaks below 2 GB per process);
    FSB_REF_PROCS caps it (tests)."""
    n = max(1, min(cpu_cores(), mem_available_bytes() // (2 << 30)))
    cap = os.environ.get("FSB_REF_PROCS")
    return min(n, max(1, int(cap))) if cap else n


def cpu_baseline_sample(name: str) -> dict:
    """Bounded CPU sample for the B200 arm (about 25 s): the oracle port solves the
    whole C3 frame with N=1 and with N=2 warps (all levels, setup included) on all
    cores; the NumPy cost is linear in N, so T(N) = T(1) + (N - 1) (T(2) - T(1))."""
    procs = max(2, cpu_procs())
    t0 = time.perf_counter()
    secs = cpu_wave("port", name, procs, warps=(1, 2))
    wall = time.perf_counter() - t0
    t1 = statistics.mean(secs[0::2])
    t2 = statistics.mean(secs[1::2])
    n = params_dict(name)["warp_iters"]
    t_frame = t1 + (n - 1) * (t2 - t1)
    fps = procs / t_frame
    return {"value": fps, "unit": "frames/s", "cores": procs, "kind": "port",
            "sample": (f"oracle/fs_oracle.py (fp64 NumPy restatement pinned to the reference) "
                       f"on {procs} host processes ({cpu_model()}): whole {name.upper()} frames "
                       f"at N=1 ({t1:.1f} s) and N=2 ({t2:.1f} s) warps, extrapolated linearly "
                       f"to N={n} ({t_frame:.0f} s per frame per core); {wall:.0f} s wall"),
            "mpix_iter_per_s": fps * pixel_iters_per_frame(name) / 1e6}


# ---------------------------------------------------------------- reference arm

def run_reference(a) -> None:
    """CPU reference arm: rank 0 only; one wave of whole frames on all host cores."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    if a.workload == "c4":
        raise SystemExit("--impl reference times single frames (c1, c2, c3, c5)")
    kind = "reference" if _reference_module() is not None else "port"
    procs = cpu_procs()
    pair = None if a.workload == "c3" else reference_pair(a.workload)
    t0 = time.perf_counter()
    secs = cpu_wave(kind, a.workload, procs, pair=pair)
    wave = time.perf_counter() - t0
    fps = procs / wave
    ppf = pixel_iters_per_frame(a.workload)
    impl = ("fisheyestereo.solve_pyramid, the unmodified reference package "
            "(baseline/_ref)" if kind == "reference" else
            "oracle/fs_oracle.pyramid_solve (pinned port; baseline/_ref absent)")
    sample = (f"{impl}: one wave of {procs} whole {a.workload.upper()} frames, one "
              f"single-threaded process "
              f"per host core ({cpu_model()}); per-frame {min(secs):.0f}-{max(secs):.0f} s, "
              f"wave {wave:.0f} s. --steps/--warmup are not applied: a frame is minutes "
              f"of NumPy with no warm-up state")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    line = {"impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s",
            "n_gpus": world, "steps": 1, "warmup": 0, "ms_per_step": wave * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic (reference-rendered {a.workload.upper()} pair, float32 values)",
            "config": config_of(a.workload, world),
            "mpix_iter_per_s": fps * ppf / 1e6,
            "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": procs, "kind": kind,
                             "sample": sample},
            "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- B200 arm

def pd32_roofline(eng, rig, prm, img0, iters=50):
    """fp32 path: time the primal-dual kernel (k_pd_tma, fsb_pd_iterate) at the
    finest level with CUDA events on its launch stream."""
    import ctypes as C
    import torch
    from paper_1909_07545_b200 import _dev, _ext
    from paper_1909_07545_b200.fields import trajectory_field_device, translation_only_rig
    from paper_1909_07545_b200.solver import _Level
    L = _ext.lib()
    H, W = rig.cam0.height, rig.cam0.width
    lv = _Level(H, W)
    lv.i0.copy_(img0)
    lv.i1.copy_(eng.i1c)
    lv.mask.copy_(eng.mask)
    d, ok = trajectory_field_device(rig.cam0, translation_only_rig(rig).pose.translation,
                                    prm.epsilon_scale)
    lv.traj.copy_(d)
    lv.traj_ok.copy_(ok)
    lv.u.zero_(); lv.wv.zero_()
    ps = _ext.params_struct(prm)
    s = _dev.scratch(L.fsb_smooth_scratch_bytes(H, W))
    st = lv.struct()
    sp = _dev.stream_ptr()
    _ext.check(L.fsb_level_setup(C.byref(st), C.byref(ps), _dev.ptr(s), s.numel(), sp), "setup")
    for t in (lv.v, lv.v_bar, lv.p, lv.q):
        t.zero_()
    lv.u_bar.copy_(lv.u)
    _ext.check(L.fsb_warp_linearize(C.byref(st), sp), "linearize")
    _ext.check(L.fsb_pd_iterate(C.byref(st), C.byref(ps), 5, None, None, sp), "pd")
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    _ext.check(L.fsb_pd_iterate(C.byref(st), C.byref(ps), iters, None, None, sp), "pd")
    e1.record(stream)
    torch.cuda.synchronize()
    t_iter = e0.elapsed_time(e1) / 1e3 / iters
    cycles = 5  # PD cycles per launch of the temporally blocked kernel (its halo)
    t_launch = t_iter * cycles
    bytes_launch = PD32_BYTES_PER_PIXEL_ITER * H * W * cycles
    peak, peak_src = measured_peak()
    achieved = bytes_launch / t_launch / 1e9
    traffic, traffic_src = profiled_traffic("*_tma_pd_ncu.txt")
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic,
            "kernel": f"k_pd_tma (persistent, TMA-fed), {cycles} PD cycles per launch",
            "algorithmic_bytes_per_launch": bytes_launch,
            "per_unit": (f"{PD32_BYTES_PER_PIXEL_ITER} B per pixel-iteration x {H}x{W} px x "
                         f"{cycles} cycles"),
            "us_per_launch": t_launch * 1e6, "us_per_pd_cycle": t_iter * 1e6,
            "peak_source": peak_src, "traffic_source": traffic_src,
            "note": ("temporal blocking keeps the state on chip for 5 cycles: algorithmic "
                     "bytes exceed the DRAM traffic (see traffic)")}


def pd64_roofline(eng, prm) -> tuple[dict, dict]:
    """float64 path: live CUDA-event timing of the finest level's primal-dual
    launches and warp prologue inside a solve on the solve stream
    (fsb_solve_pyramid_f64_timed); returns (PD roofline, prologue roofline)."""
    eng.time_phases(0)  # warm
    t = eng.time_phases(0)
    H, W = t["h"], t["w"]
    launches = t["warps"] * t["pd_launches_per_warp"]
    cycles = prm.pd_iters / t["pd_launches_per_warp"]
    us_launch = t["pd_ms"] * 1e3 / launches
    bytes_launch = PD64_BYTES_PER_PIXEL_ITER * H * W * cycles
    peak, peak_src = measured_peak()
    achieved = bytes_launch / (us_launch * 1e-6) / 1e9
    traffic, traffic_src = profiled_traffic("*_pd64_ncu.txt")
    pd = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
          "frac": achieved / peak, "traffic": traffic,
          # the real DRAM fraction: ncu bytes of one launch over the live launch time
          "dram_frac": (traffic / (us_launch * 1e-6) / 1e9 / peak) if traffic else None,
          "kernel": (f"float64 primal-dual launch at the finest level ({W}x{H}), "
                     f"{cycles:g} PD cycles per launch"),
          "algorithmic_bytes_per_launch": bytes_launch,
          "per_unit": (f"{PD64_BYTES_PER_PIXEL_ITER} B per pixel-iteration (float64 state and "
                       f"constants) x {H}x{W} px x {cycles:g} cycles"),
          "us_per_launch": us_launch, "us_per_pd_cycle": us_launch / cycles,
          "launches_timed": launches,
          "timer": "CUDA events on the solve stream around each warp's PD launches "
                   "(fsb_solve_pyramid_f64_timed)",
          "peak_source": peak_src, "traffic_source": traffic_src}
    us_warp = t["sample_ms"] * 1e3 / t["warps"]
    pbytes = PRO64_BYTES_PER_PIXEL_WARP * H * W
    pa = pbytes / (us_warp * 1e-6) / 1e9
    ptraffic, ptraffic_src = profiled_traffic("*_pro64_ncu.txt")
    pro = {"bound": "hbm", "achieved": pa, "peak": peak, "unit": "GB/s", "frac": pa / peak,
           "traffic": ptraffic, "traffic_source": ptraffic_src,
           "kernel": f"float64 warp prologue (sample + linearise) at {W}x{H}",
           "algorithmic_bytes_per_launch": pbytes,
           "per_unit": f"{PRO64_BYTES_PER_PIXEL_WARP} B per pixel per warp x {H}x{W} px",
           "us_per_warp": us_warp}
    return pd, pro


def parity_vs_reference(u: np.ndarray, mask: np.ndarray) -> dict | None:
    """|u - u_reference| on the reference's solve mask (tests/golden/c3_solution.npz)."""
    if not C3_SOLUTION.exists():
        return None
    with np.load(C3_SOLUTION) as z:
        ur, mr = z["u"].astype(np.float64), z["mask"]
    e = np.abs(np.asarray(u, np.float64) - ur)[mr]
    return {"median": float(np.median(e)), "p99": float(np.percentile(e, 99)),
            "max": float(e.max()), "mask_identical": bool(np.array_equal(mask, mr)),
            "gate": "median <= 1e-3 px, p99 <= 1e-2 px (north star)",
            "pass": bool(np.median(e) <= 1e-3 and np.percentile(e, 99) <= 1e-2)}


def _graph_fps(eng, K, warmup, stream, flush, world, dist) -> tuple[float, object]:
    """K timed graph replays (events on the launch stream, L2 flushed between)."""
    import torch
    for _ in range(max(warmup, 0)):
        eng.replay()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(K)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(torch.cuda.current_device())
    with clk:
        for k in range(K):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            ev[k][0].record(stream)
            eng.replay()
            ev[k][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_ms = sum(s.elapsed_time(e) for s, e in ev)
    t_all = torch.tensor([t_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t_all, op=dist.ReduceOp.MAX)
    return float(t_all.item()) / 1e3, clk


def _e2e(solve, h0, h1, K, warmup, world, dist) -> tuple[float, list]:
    """Seconds for K calls of the public API on host float64 arrays (max over
    ranks), and the per-call milliseconds of this rank."""
    import torch
    for _ in range(max(warmup, 10)):  # engine build, graph capture, pinned pools
        res = solve(h0, h1)
    del res
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    calls = []
    t0 = time.perf_counter()
    for _ in range(K):
        t1 = time.perf_counter()
        res = solve(h0, h1)  # returns after its D2H: the call is synchronous
        calls.append((time.perf_counter() - t1) * 1e3)
    torch.cuda.synchronize()
    te = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    return float(te.item()), calls


def run_b200(a) -> None:
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_1909_07545_b200 import synth as S
    from paper_1909_07545_b200.solver import Solver, solve_pyramid

    name = a.workload
    rig, prm = product_rig(name), product_params(name)
    H, W = rig.cam0.height, rig.cam0.width
    if name == "c3":
        h0, h1 = load_c3_pair()
        img0 = torch.from_numpy(h0).cuda()
        img1 = torch.from_numpy(h1).cuda()
    else:  # every rank solves its own frame: the scene is reseeded per rank
        ss = WORKLOADS[name]["ss"]
        scene = S.reseed_scene(S.default_scene(), rank)
        img0 = S.render_device(scene, rig.cam0, supersample=ss)[0]
        img1 = S.render_device(scene, rig.cam1, pose=rig.pose, supersample=ss)[0]
        h0, h1 = img0.cpu().numpy(), img1.cpu().numpy()
    # host float64 arrays holding the float32 input values (the API's input type)
    x0, x1 = h0.astype(np.float64), h1.astype(np.float64)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    K = a.steps
    ppf = pixel_iters_per_frame(name)

    # ---- the credited path: float64 (drop-in default), graph replay, inputs in HBM
    eng = Solver(rig, prm, precision="fp64")
    eng.i0.copy_(img0)
    eng.i1.copy_(img1)
    kernels = eng.capture()
    t_max, clk = _graph_fps(eng, K, a.warmup, stream, flush, world, dist)
    fps = world * K / t_max
    parity = parity_vs_reference(eng.u.cpu().numpy(), eng.mask.cpu().numpy().astype(bool)) \
        if (name == "c3" and rank == 0) else None

    e2e = None
    if not a.no_e2e:
        te, calls = _e2e(lambda p, q: solve_pyramid(p, q, rig, prm), x0, x1, K, a.warmup,
                         world, dist)
        e2e = {"value": world * K / te, "unit": "frames/s",
               "ms_per_call": {"min": min(calls), "median": statistics.median(calls),
                               "max": max(calls), "argmax": calls.index(max(calls))},
               "h2d_bytes_per_step": 2 * H * W * 8,
               "d2h_bytes_per_step": H * W * (8 + 16 + 16 + 1 + 8),
               "api": "paper_1909_07545_b200.solve_pyramid (float64 host arrays in, "
                      "StereoResult of float64 / bool host arrays out; default precision)",
               "timer": "host wall clock around each API call: host copy into pinned "
                        "staging, H2D of i0 / i1 (float64), graph replay, D2H of u, w, v "
                        "after the frame and of mask, i1_calibrated during it (side stream "
                        "behind the graph's early-output event) into pinned output buffers"}
    roof = pro = None
    if rank == 0:
        roof, pro = pd64_roofline(eng, prm)
    del eng

    # ---- the float32 path (secondary): faster, misses the p99 gate at N=50
    fp32 = None
    if rank == 0 and not a.no_fp32:
        e32 = Solver(rig, prm, precision="fp32")
        e32.i0.copy_(img0)
        e32.i1.copy_(img1)
        e32.capture()
        t32, _ = _graph_fps(e32, K, a.warmup, stream, flush, 1, None)
        fp32 = {"value": K / t32, "unit": "frames/s", "dtype": "f32",
                "parity_vs_reference": (parity_vs_reference(
                    e32.u.cpu().numpy(), e32.mask.cpu().numpy().astype(bool))
                    if name == "c3" else None)}
        if not a.no_e2e:
            te, _ = _e2e(lambda p, q: solve_pyramid(p, q, rig, prm, precision="fp32"), x0, x1,
                         K, a.warmup, 1, None)
            fp32["e2e"] = {"value": K / te, "unit": "frames/s",
                           "h2d_bytes_per_step": 2 * H * W * 4,
                           "d2h_bytes_per_step": H * W * (8 + 16 + 16 + 1 + 8)}
        fp32["roofline"] = pd32_roofline(e32, rig, prm, img0)
        del e32

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu and name == "c3":
        cpu = cpu_baseline_sample(name)

    if rank == 0:
        line = {
            "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world, "steps": K,
            "warmup": a.warmup, "ms_per_step": t_max * 1e3 / K, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": ("synthetic (reference-rendered C3 pair, float32 values)" if name == "c3"
                     else "synthetic (GPU ray-cast default_scene, reseeded per rank)"),
            "config": config_of(name, world),
            "mpix_iter_per_s": fps * ppf / 1e6,
            "e2e": e2e,
            "gpu_launches": kernels * K,
            "kernels_per_frame": kernels,
            "roofline": roof,
            "roofline_prologue": pro,
            "parity_vs_reference": parity,
            "fp32_path": fp32,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_sequence(a) -> None:
    """C4: each rank solves its contiguous block of the 256-frame sequence, one
    frame per stream per step (pose and scene differ per frame; no data-path
    collective)."""
    import torch
    import torch.distributed as dist
    from paper_1909_07545_b200 import _ext
    from paper_1909_07545_b200 import synth as S
    from paper_1909_07545_b200.sequence import c4_rig, max_over_ranks, partition
    from paper_1909_07545_b200.solver import Solver

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    prm = product_params("c4")
    ss = WORKLOADS["c4"]["ss"]
    block = list(partition(256, world, rank))
    K, Wm = a.steps, max(a.warmup, 0)
    B = max(1, a.streams)  # frames in flight per GPU, one engine + stream each
    frames = [block[k % len(block)] for k in range((Wm + K) * B)]
    base = S.default_scene()
    imgs = []
    for i in frames:  # inputs rendered before timing, resident in HBM
        rig = c4_rig(i)
        sc = S.reseed_scene(base, i)
        imgs.append((rig, S.render_device(sc, rig.cam0, supersample=ss)[0].double(),
                     S.render_device(sc, rig.cam1, pose=rig.pose, supersample=ss)[0].double()))
    engs = [Solver(imgs[0][0], prm, precision=a.precision) for _ in range(B)]
    streams = [torch.cuda.Stream() for _ in range(B)]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    dt = torch.float64 if a.precision == "fp64" else torch.float32

    def step(k):
        ready = torch.cuda.Event()
        ready.record(stream)
        done = []
        for b in range(B):
            rig, i0, i1 = imgs[(k * B + b) % len(imgs)]
            with torch.cuda.stream(streams[b]):
                streams[b].wait_event(ready)
                engs[b].rs = _ext.rig_struct(rig)  # per-frame pose; same shapes, same workspace
                engs[b].run(i0.to(dt), i1.to(dt))
                e = torch.cuda.Event()
                e.record(streams[b])
                done.append(e)
        for e in done:
            stream.wait_event(e)

    for k in range(Wm):
        step(k)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(K)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(K):
            flush.zero_()
            ev[k][0].record(stream)
            step(Wm + k)
            ev[k][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_max = max_over_ranks(sum(s_.elapsed_time(e) for s_, e in ev) / 1e3, device="cuda")
    fps = world * K * B / t_max
    ppf = pixel_iters_per_frame("c4")
    if rank == 0:
        cfg = config_of("c4", world)
        cfg.update(frames_per_step_per_gpu=B, streams_per_gpu=B, frames_per_rank=len(block))
        print(json.dumps({
            "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world, "steps": K,
            "warmup": a.warmup, "ms_per_step": t_max * 1e3 / K, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "f64" if a.precision == "fp64" else "f32",
            "data": "synthetic (GPU ray-cast default_scene reseeded per frame, ss=1)",
            "config": cfg, "mpix_iter_per_s": fps * ppf / 1e6, "e2e": None,
            "gpu_launches": None, "roofline": None, "cpu_baseline": None,
            "clocks": clk.summary()}), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------- launcher

def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch(argv: list, n: int) -> int:
    """Re-exec this script as n ranks under torch.distributed.run (one per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), str(Path(__file__).resolve()), *argv]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "4"))
    return subprocess.call(cmd, env=env)


def run_launch_check(a) -> None:
    """No-GPU launcher check (tests/test_bench_launch.py): forms the process
    group over gloo, times a stub step, reduces the max over ranks."""
    import torch.distributed as dist
    from paper_1909_07545_b200.sequence import max_over_ranks
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        dist.init_process_group("gloo")
    t = max_over_ranks(0.01 * (rank + 1))
    if rank == 0:
        print(json.dumps({"impl": "launch-check", "n_gpus": world, "steps": a.steps,
                          "t_max": t}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main(argv=None) -> int:
    argv = sys.argv[1:] if argv is None else list(argv)
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c3")
    ap.add_argument("--precision", choices=["fp64", "fp32"], default="fp64",
                    help="C4 sequence path precision")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-fp32", action="store_true", help="skip the secondary fp32 legs")
    ap.add_argument("--streams", type=int, default=1,
                    help="C4: frames in flight per GPU (one engine and CUDA stream each)")
    ap.add_argument("--no-e2e", action="store_true", help="skip the public-API e2e legs")
    ap.add_argument("--launch-check", action="store_true", help=argparse.SUPPRESS)
    a = ap.parse_args(argv)
    if a.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if a.impl == "reference":
        run_reference(a)
        return 0
    if "WORLD_SIZE" not in os.environ and a.gpus > 1:
        return relaunch(argv, a.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}")
    if a.launch_check:
        run_launch_check(a)
    elif a.workload == "c4":
        run_sequence(a)
    else:
        run_b200(a)
    return 0


if __name__ == "__main__":
    sys.exit(main())
