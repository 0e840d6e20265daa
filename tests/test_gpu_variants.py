"""The float64 path's kernel variants agree (each switch is read once per
process, so every variant runs in a child process on the golden pair and on a
C1 frame, the C1 frame also with diagnostics: the DIAG kernel variants). The
default at these sizes (k64_level on the levels that fit one cluster — the
golden pair, C1 80^2 — k64_tile over the per-level work lists elsewhere,
phase-staggered persistent schedule, NaN-texel prologue on small levels) against
  * k64_tile everywhere (FSB_PD64K=tilel)                  -> bit-identical,
  * the non-persistent schedule (FSB_PD64_PERSIST=0)      -> bit-identical,
  * per-level setup on the caller's stream (FSB_OVERLAP=0) -> bit-identical,
  * k64_tile over every tile with masked loads (FSB_PD64K=tile; also the
    per-warp launches on the small levels)                -> <= 1e-10 px,
  * the k64_ctile cluster regions on the halo-2 levels, as the default uses
    them from 512^2 up (FSB_CTILE_MIN=1), in four cluster shapes / halos, and
    the TMA-fed k64_tma (FSB_PD64K=tma)                   -> <= 1e-10 px (they
    differ only in where the compiler contracts a multiply-add, ~1e-13 px),
  * the per-warp launches instead of the whole-level cluster kernel on the
    levels that fit one cluster (FSB_LEVEL64=0)           -> <= 1e-10 px,
  * the masked-gather prologue everywhere (FSB_PRO64=old) -> <= 1e-10 px,
  * the round-1 k64_block, no FMA (FSB_PD64K=block)       -> <= 1e-8 px.
Scheduling and load strategy must not change a single bit of the answer."""

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
from conftest import load_golden
import test_gpu_solve as T
import bench
from paper_1909_07545_b200 import synth as S
from paper_1909_07545_b200.solver import solve_pyramid
g = load_golden("pyramid_solve")
r = solve_pyramid(g["i0"], g["i1"], T._rig(g), T._params(g))
rig1, prm1 = bench.product_rig("c1"), bench.product_params("c1")
sc = S.default_scene()
i0 = S.render(sc, rig1.cam0, supersample=1)[0]
i1 = S.render(sc, rig1.cam1, pose=rig1.pose, supersample=1)[0]
r1 = solve_pyramid(i0, i1, rig1, prm1)
d = solve_pyramid(i0, i1, rig1, prm1, collect_diagnostics=True).diagnostics
np.savez(sys.argv[2], u=r.u, w=r.w, v=r.v, u1=r1.u, w1=r1.w,
         d_p=np.array(d.max_p_norm), d_q=np.array(d.max_q_norm), d_du=np.array(d.max_du),
         d_mean=np.array(d.mean_abs_du))
"""


def _run(tmp_path, name, env_extra):
    out = tmp_path / f"{name}.npz"
    env = dict(os.environ, **env_extra)
    subprocess.run([sys.executable, "-c", _CHILD, str(ROOT), str(out)], env=env, check=True,
                   timeout=900)
    with np.load(out) as z:
        return {k: z[k] for k in z.files}


@pytest.mark.parametrize("name,env,tol", [
    ("tilel", {"FSB_PD64K": "tilel"}, 0.0),
    ("ctile", {"FSB_CTILE_MIN": "1"}, 1e-10),
    ("ctile_5_2_4_16", {"FSB_CTILE_MIN": "1", "FSB_CTILE": "5,2,4,16"}, 1e-10),
    ("ctile_5_4_4", {"FSB_CTILE_MIN": "1", "FSB_CTILE": "5,4,4"}, 1e-10),
    ("ctile_10_4_4", {"FSB_CTILE_MIN": "1", "FSB_CTILE": "10,4,4"}, 1e-10),
    ("tma", {"FSB_PD64K": "tma"}, 1e-10),
    ("persist0", {"FSB_PD64_PERSIST": "0"}, 0.0),
    ("no_overlap", {"FSB_OVERLAP": "0"}, 0.0),
    ("alltiles", {"FSB_PD64K": "tile"}, 1e-10),
    ("level_off", {"FSB_LEVEL64": "0"}, 1e-10),
    ("prologue_old", {"FSB_PRO64": "old"}, 1e-10),
    ("block", {"FSB_PD64K": "block"}, 1e-8),
])
def test_float64_kernel_variants_agree(tmp_path, name, env, tol):
    base = _run(tmp_path, "default", {})
    var = _run(tmp_path, name, env)
    for k in base:
        if k.startswith("d_"):  # diagnostics (the DIAG kernel variants): max / mean traces
            if tol == 0.0:
                assert np.array_equal(base[k], var[k]), (name, k)
            else:
                assert np.allclose(base[k], var[k], rtol=1e-6, atol=1e-12), (name, k)
            continue
        d = float(np.max(np.abs(base[k] - var[k])))
        assert d <= tol, (name, k, d)
