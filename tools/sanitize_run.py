"""Small solves that exercise every hot kernel, for compute-sanitizer runs
(tools/sanitize.sh): C3 geometry with N=1 warp (1024^2 .. 64^2 levels:
k_pd_tma on the large levels, the 16-CTA cluster kernel k_level_cluster on
64^2 / 128^2, the fp64 k64_tile / NaN-texel prologue), and C1 (320^2
equidistant, N=2). argv[1] = fp32 | fp64 | both."""
import sys
from dataclasses import replace
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import bench
from paper_1909_07545_b200.solver import solve_pyramid

which = sys.argv[1] if len(sys.argv) > 1 else "both"
precs = ["fp32", "fp64"] if which == "both" else [which]
h0, h1 = bench.load_c3_pair()
rig = bench.product_rig("c3")
prm = replace(bench.product_params("c3"), warp_iters=1)
for p in precs:
    r = solve_pyramid(h0.astype(np.float64), h1.astype(np.float64), rig, prm, precision=p,
                      collect_diagnostics=True)
    assert np.isfinite(r.u).all()
rig1, prm1 = bench.product_rig("c1"), replace(bench.product_params("c1"), warp_iters=2)
from paper_1909_07545_b200 import synth as S
sc = S.default_scene()
i0 = S.render(sc, rig1.cam0, supersample=1)[0]
i1 = S.render(sc, rig1.cam1, pose=rig1.pose, supersample=1)[0]
for p in precs:
    r = solve_pyramid(i0, i1, rig1, prm1, precision=p)
    assert np.isfinite(r.u).all()
torch.cuda.synchronize()
print("sanitize_run ok", precs)
