"""Generate the C3 headline-config fixtures by running the REFERENCE implementation.

TEST INFRASTRUCTURE ONLY. Run in the build container (the reference is not on
the GPU box):

    python oracle/make_c3_fixture.py        # reads /root/reference/pkg/src, ~12 min

Writes
  tests/golden/c3_pair.npz      the C3 input pair (BASELINE config 3):
                                reference `synth.render(default_scene(), ...,
                                supersample=2)` of the 1024^2 unified rig under the
                                6-DoF pose, rounded to float32 (the dtype the B200
                                path and both bench arms consume);
  tests/golden/c3_solution.npz  the reference's own `solve_pyramid` (solver.py:
                                401-452, SolverParams() defaults: N=50, K=10, 5
                                levels) on exactly those float32 values (upcast to
                                float64): u (float32-rounded), mask,
                                i1_calibrated (float32-rounded), and the wall time.

tests/test_gpu_c3_parity.py gates both GPU paths against c3_solution.npz at full
size; bench.py feeds c3_pair.npz to the B200 arm and to the reference arm.
"""

from __future__ import annotations

import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def c3_rig(camera):
    """BASELINE config 3."""
    cam = camera.UnifiedCamera(width=1024, height=1024, fx=455.0, fy=455.0, cx=511.5,
                               cy=511.5, fov=np.pi, xi=0.9)
    pose = camera.RelativePose.from_displacement((0.08, 0.02, 0.03),
                                                 rotvec=(0.01, 0.03, -0.02))
    return camera.StereoRig(cam, cam, pose)


def _render(which: int) -> np.ndarray:
    sys.path.insert(0, str(REF))
    from fisheyestereo import camera, synth
    rig = c3_rig(camera)
    scene = synth.default_scene()
    if which == 0:
        img = synth.render(scene, rig.cam0, supersample=2)[0]
    else:
        img = synth.render(scene, rig.cam1, pose=rig.pose, supersample=2)[0]
    return np.asarray(img, np.float32)


def main() -> int:
    sys.path.insert(0, str(REF))
    from fisheyestereo import camera, solver
    OUT.mkdir(parents=True, exist_ok=True)
    pair = OUT / "c3_pair.npz"
    if pair.exists():
        d = np.load(pair)
        i0, i1 = d["i0"], d["i1"]
    else:
        t0 = time.time()
        with ProcessPoolExecutor(2) as ex:
            i0, i1 = ex.map(_render, (0, 1))
        print(f"rendered C3 pair in {time.time() - t0:.0f} s", flush=True)
        np.savez_compressed(pair, i0=i0, i1=i1)
    rig = c3_rig(camera)
    t0 = time.time()
    res = solver.solve_pyramid(i0.astype(np.float64), i1.astype(np.float64), rig,
                               solver.SolverParams())
    dt = time.time() - t0
    print(f"reference solve_pyramid C3: {dt:.0f} s on 1 core", flush=True)
    np.savez_compressed(OUT / "c3_solution.npz", u=res.u.astype(np.float32), mask=res.mask,
                        i1c=res.i1_calibrated.astype(np.float32),
                        seconds=np.float64(dt))
    return 0


if __name__ == "__main__":
    sys.exit(main())
