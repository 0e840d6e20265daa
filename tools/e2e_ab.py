"""A/B of the public-API download on C3: fp32 chunked D2H + host widening
(current) vs float64 widening on the device + full-size D2H (previous)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import bench
from paper_1909_07545_b200 import synth as S
from paper_1909_07545_b200.solver import Solver, solve_pyramid, _CACHE

rig, prm, desc, ss = bench.workload("c3")
sc = S.default_scene()
i0 = S.render_device(sc, rig.cam0, supersample=ss)[0].cpu().numpy().astype(np.float64)
i1 = S.render_device(sc, rig.cam1, pose=rig.pose, supersample=ss)[0].cpu().numpy().astype(np.float64)
new = Solver._download_widened


def old(self, st):
    for k, dt in self._OUT:
        st[k][0].copy_(getattr(self, k).to(dt), non_blocking=True)
    torch.cuda.current_stream().synchronize()


ref = None
for _ in range(5):
    r = solve_pyramid(i0, i1, rig, prm)
res = {"new": [], "old": []}
for rep in range(4):
    for name, fn in (("old", old), ("new", new)):
        Solver._download_widened = fn
        t0 = time.perf_counter()
        for _ in range(20):
            r = solve_pyramid(i0, i1, rig, prm)
        res[name].append((time.perf_counter() - t0) / 20 * 1e3)
        if ref is None:
            ref = {k: getattr(r, k).copy() for k in ("u", "w", "v", "mask", "i1_calibrated")}
        else:
            for k, a in ref.items():
                assert np.array_equal(a, getattr(r, k)), k
Solver._download_widened = new
print({k: [round(x, 3) for x in v] for k, v in res.items()}, "ms/call; outputs bit-identical")
