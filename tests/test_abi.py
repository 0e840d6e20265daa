"""C-ABI checks that need no GPU: the library loads and exports exactly what
include/fsb200.h declares; host-only entry points behave like the reference."""

import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def header_symbols():
    text = (ROOT / "include" / "fsb200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char\*|void\*)\s+(fsb_\w+)\(", text, re.M)))


def test_header_matches_binding_list():
    from paper_1909_07545_b200 import _ext
    assert header_symbols() == sorted(_ext.EXPORTED)


def test_library_exports_every_header_symbol():
    from paper_1909_07545_b200 import _ext
    L = _ext.lib()
    missing = [s for s in header_symbols() if not hasattr(L, s)]
    assert not missing
    assert L.fsb_version().startswith(b"fsb200")


def test_pyramid_shapes_host_entry():
    from paper_1909_07545_b200.rasters import pyramid_shapes
    # rasters.py:207-221 known answers (reference test_rasters.py:133-162)
    assert [w for _, w in pyramid_shapes(800, 800, 5, 2.0, 50)] == [800, 400, 200, 100, 50]
    assert [w for _, w in pyramid_shapes(120, 120, 5, 2.0, 50)] == [120, 60]
    assert [w for _, w in pyramid_shapes(64, 64, 3, 2.0, 8)] == [64, 32, 16]
    # survey §0-3: C2 (640x480, 5 levels) needs min_width 40; C5 needs 32
    assert len(pyramid_shapes(480, 640, 5, 2.0, 40)) == 5
    assert len(pyramid_shapes(2048, 2048, 7, 2.0, 32)) == 7
    for levels, scale in [(0, 2.0), (3, 1.0), (3, 0.5)]:
        with pytest.raises(ValueError):
            pyramid_shapes(64, 64, levels, scale, 8)


def test_workspace_and_diag_counts():
    import ctypes as C
    from paper_1909_07545_b200 import _ext
    from paper_1909_07545_b200.camera import RelativePose, StereoRig, UnifiedCamera
    from paper_1909_07545_b200.solver import SolverParams
    L = _ext.lib()
    cam = UnifiedCamera(width=1024, height=1024, fx=455.0, fy=455.0, cx=511.5, cy=511.5,
                        fov=3.141592653589793, xi=0.9)
    rig = StereoRig(cam, cam, RelativePose.from_displacement((0.08, 0.02, 0.03),
                                                             rotvec=(0.01, 0.03, -0.02)))
    rs, ps = _ext.rig_struct(rig), _ext.params_struct(SolverParams())
    nbytes = L.fsb_solve_pyramid_workspace_bytes(C.byref(rs), C.byref(ps))
    assert 100e6 < nbytes < 1e9  # ~ 0.25 KB/px of resident state at 1024^2
    npd, nw = C.c_int64(), C.c_int64()
    assert L.fsb_diag_counts(1024, 1024, C.byref(ps), C.byref(npd), C.byref(nw)) == 5
    assert npd.value == 5 * 50 * 10 and nw.value == 5 * 50
    bad = _ext.params_struct(SolverParams())
    bad.du_max = 0.0
    assert L.fsb_solve_pyramid_workspace_bytes(C.byref(rs), C.byref(bad)) == 0


def test_params_validation_mirrors_reference():
    from paper_1909_07545_b200.solver import SolverParams
    with pytest.raises(ValueError):
        SolverParams(lam=-1.0)
    with pytest.raises(ValueError):
        SolverParams(du_max=0.0)
    with pytest.raises(ValueError):
        SolverParams(warp_iters=0)
    with pytest.raises(ValueError):
        SolverParams.from_dict({"lambda_weight": 1.0})
    assert SolverParams.from_dict(SolverParams().to_dict()) == SolverParams()


def test_no_cpu_fallback_without_device(monkeypatch):
    import torch
    from paper_1909_07545_b200 import _dev
    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _dev.device()


def test_product_never_imports_oracle():
    pkg = ROOT / "paper_1909_07545_b200"
    for f in pkg.rglob("*.py"):
        assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", f.read_text(), re.M), f


def test_binding_arity_matches_header():
    """Every ctypes signature in _ext.py takes as many arguments as the C
    declaration in include/fsb200.h (a short binding passes garbage for the
    missing trailing arguments)."""
    from paper_1909_07545_b200 import _ext
    L = _ext.lib()
    text = (ROOT / "include" / "fsb200.h").read_text()
    decls = re.findall(r"^\s*(?:int|size_t|const char\*|void\*)\s+(fsb_\w+)\(([^;]*)\);",
                       text, re.M | re.S)
    assert len(decls) == len(header_symbols())
    bad = []
    for name, args in decls:
        args = " ".join(args.split())
        n = 0 if args in ("", "void") else args.count(",") + 1
        f = getattr(L, name)
        if f.argtypes is None or len(f.argtypes) != n:
            bad.append((name, n, None if f.argtypes is None else len(f.argtypes)))
    assert not bad, bad
