"""Host-side API (no GPU): the rig JSON schema round-trips against the
reference's own rig_to_dict output (tests/golden/rig_json.npz), and the
parameter dataclass keeps the reference's strictness."""

import json

import numpy as np
import pytest

from conftest import load_golden


def test_rig_json_matches_reference_schema(tmp_path):
    from paper_1909_07545_b200.camera import load_rig, rig_from_dict, rig_to_dict, save_rig
    for rec in load_golden("rig_json")["rigs"]:
        d = json.loads(str(rec))
        rig = rig_from_dict(d)
        again = rig_to_dict(rig)
        assert json.dumps(again, sort_keys=True) == json.dumps(d, sort_keys=True)
        save_rig(tmp_path / "rig.json", rig)
        back = load_rig(tmp_path / "rig.json")
        np.testing.assert_array_equal(back.pose.rotation, rig.pose.rotation)
        np.testing.assert_array_equal(back.pose.translation, rig.pose.translation)
        assert back.cam0.model == rig.cam0.model and back.cam1.model == rig.cam1.model


def test_solver_params_strict_from_dict():
    from paper_1909_07545_b200.solver import SolverParams
    p = SolverParams.from_dict({"warp_iters": 7, "lam": 3.0})
    assert p.warp_iters == 7 and p.lam == 3.0 and p.pd_iters == 10
    with pytest.raises(ValueError):
        SolverParams.from_dict({"warp_iterations": 7})
    with pytest.raises(ValueError):
        SolverParams(alpha0=0.0)
    with pytest.raises(ValueError):
        SolverParams(du_max=-1.0)
    with pytest.raises(ValueError):
        SolverParams(pd_iters=0)
    assert SolverParams.from_dict(p.to_dict()) == p


def test_engine_cache_checkout_is_exclusive(monkeypatch):
    """solve_pyramid's engine cache (no GPU: the engine is stubbed): an engine
    is never used by two threads at once, concurrent same-rig callers get
    their own engines and those engines are kept (a bounded idle list per
    key) and reused, the cache keeps at most _CACHE_KEYS keys, and an engine
    whose call raised is released instead of returned."""
    import threading
    import time
    from paper_1909_07545_b200 import solver as SV
    from paper_1909_07545_b200.camera import RelativePose, StereoRig, UnifiedCamera

    made, clash, released = [], [], []

    class FakeSolver:
        def __init__(self, rig, params, diag=False, precision="fp64"):
            self.busy = threading.Lock()
            self.fail = False
            made.append(self)

        def solve(self, i0, i1):
            if not self.busy.acquire(blocking=False):
                clash.append(self)
                return None
            try:
                time.sleep(0.002)
                if i0 is BOOM:
                    raise RuntimeError("CUDA error during replay")
                return self
            finally:
                self.busy.release()

        def release(self):
            released.append(self)

    monkeypatch.setattr(SV, "Solver", FakeSolver)
    monkeypatch.setattr(SV, "_CACHE", SV.OrderedDict())
    cam = UnifiedCamera(width=8, height=6, fx=4.0, fy=4.0, cx=3.5, cy=2.5, fov=np.pi, xi=0.9)

    def rig(k):
        return StereoRig(cam, cam, RelativePose.from_displacement((0.1 + 0.01 * k, 0, 0)))

    img = np.zeros((6, 8))
    BOOM = np.zeros((6, 8))
    prm = SV.SolverParams()

    def work(t, n=20):
        for k in range(n):
            SV.solve_pyramid(img, img, rig((t + k) % 6 if t % 2 else 0), prm)

    th = [threading.Thread(target=work, args=(t,)) for t in range(6)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not clash
    assert len(SV._CACHE) <= SV._CACHE_KEYS
    assert all(len(v) <= SV._CACHE_IDLE for v in SV._CACHE.values())
    # concurrent callers of ONE rig: their engines are kept and reused, so the
    # number of engines stays at the peak concurrency instead of growing per round
    monkeypatch.setattr(SV, "_CACHE", SV.OrderedDict())
    made.clear()
    for _ in range(5):
        th = [threading.Thread(target=work, args=(0, 3)) for _ in range(3)]
        for t in th:
            t.start()
        for t in th:
            t.join()
    assert len(made) <= 3, len(made)
    # serial reuse: the same rig twice in a row hits the cached engine
    a = SV.solve_pyramid(img, img, rig(0), prm)
    assert SV.solve_pyramid(img, img, rig(0), prm) is a
    # a failed call releases its engine and does not put it back
    with pytest.raises(RuntimeError):
        SV.solve_pyramid(BOOM, img, rig(0), prm)
    assert released and released[-1] is a
    assert all(e is not a for v in SV._CACHE.values() for e in v)
