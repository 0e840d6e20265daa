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
