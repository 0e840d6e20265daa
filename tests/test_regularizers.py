"""TV-L1 / Huber-TV regulariser variants (BASELINE config C5).

The reference is TGV only, so these variants are PARITY UNPINNED against it;
they are pinned against the oracle's restatement of the same update rules
(oracle/fs_oracle.py pd_cycle / step_sizes), and validated by invariants: v and
q stay exactly zero, the duals stay in the unit ball, the Huber dual is the
TV dual shrunk by 1 / (1 + sigma_p alpha1 eps), and (GPU tests) the energy
decreases from the zero initialisation as in test_solver.py:408-417."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import fs_oracle as O


def _prm(**kw):
    from paper_1909_07545_b200.solver import SolverParams
    return SolverParams(**kw)


def test_params_validate_regularizer():
    with pytest.raises(ValueError):
        _prm(regularizer="l2")
    with pytest.raises(ValueError):
        _prm(regularizer="huber", huber_eps=0.0)
    p = _prm(regularizer="huber", huber_eps=0.02)
    assert p.to_dict()["regularizer"] == "huber"


@pytest.mark.parametrize("reg", ["tv", "huber"])
def test_oracle_variant_invariants(reg):
    g = load_golden("pd")
    prm = _prm(regularizer=reg, huber_eps=0.05)
    mask = g["mask"]
    T = g["T"]
    st = O.step_sizes(T, mask, prm.alpha0, prm.alpha1, reg)
    assert st.sigma_q == 0.0 and not st.tau_v.any()
    h, w = mask.shape
    rng = np.random.default_rng(3)
    s = O.PDState(u=rng.normal(size=(h, w)), v=np.zeros((h, w, 2)), p=np.zeros((h, w, 2)),
                  q=np.zeros((h, w, 4)), u_bar=rng.normal(size=(h, w)), v_bar=np.zeros((h, w, 2)))
    iu = rng.normal(size=(h, w)) * 0.1
    rho0 = rng.normal(size=(h, w)) * 0.05
    for _ in range(6):
        s = O.pd_cycle(s, T, iu, rho0, s.u.copy(), prm, mask, st)
        assert not s.v.any() and not s.q.any() and not s.v_bar.any()
        assert np.linalg.norm(s.p, axis=-1).max() <= 1.0 + 1e-12
    if reg == "huber":
        # one dual step from p = 0: the TV step shrunk by 1 / (1 + sp eps) before projection
        sp = st.sigma_p * prm.alpha1
        p_tv = sp[..., None] * O.apply_T(T, O.grad_fwd(s.u_bar, mask))
        one = O.pd_cycle(O.PDState(u=s.u, v=s.v, p=np.zeros_like(s.p), q=s.q, u_bar=s.u_bar,
                                   v_bar=s.v_bar), T, iu, rho0, s.u, prm, mask, st)
        exp = O._unit_ball(p_tv / (1.0 + sp * prm.huber_eps)[..., None])
        np.testing.assert_allclose(one.p, exp, rtol=1e-12, atol=1e-15)
