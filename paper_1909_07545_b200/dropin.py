"""Route the reference package's own solve through the B200 path.

    import paper_1909_07545_b200.dropin as dropin
    dropin.install()      # fisheyestereo.solve_pyramid -> sm_100a kernels

The reference has no plugin layer: its callers reach the solve through the
module attribute `fisheyestereo.solver.solve_pyramid` (cli.py:153 and :240
call `solver.solve_pyramid`) or through names bound at import time
(`from fisheyestereo.solver import solve_pyramid` in its tests, and the
package re-export, __init__.py:8,16). `install()` rebinds the module
attributes, so every caller that imports after it — the CLI, the
walkthrough, the reference's own test modules — runs on the GPU with its
own `StereoRig` / `SolverParams` objects (duck-typed by the drop-in) and gets
a `StereoResult` with the same fields.

`pytest -p paper_1909_07545_b200.dropin` installs it before the test modules
are collected (tests/test_gpu_reference_dropin.py runs the reference's tests
this way) and writes the number of GPU solves to $FSB_DROPIN_COUNT at exit.
"""

from __future__ import annotations

import os
import threading

_calls = 0
_lock = threading.Lock()
_original = None


def install(precision: str = "fp64") -> None:
    """Rebind fisheyestereo.solve_pyramid / fisheyestereo.solver.solve_pyramid."""
    global _original
    import fisheyestereo
    import fisheyestereo.solver as ref_solver

    from .solver import solve_pyramid as b200_solve

    def solve_pyramid(i0, i1, rig, params, collect_diagnostics=False, traj_override=None):
        global _calls
        with _lock:
            _calls += 1
        return b200_solve(i0, i1, rig, params, collect_diagnostics, traj_override,
                          precision=precision)

    solve_pyramid.__doc__ = b200_solve.__doc__
    solve_pyramid.__wrapped__ = b200_solve
    if _original is None:
        _original = ref_solver.solve_pyramid
    ref_solver.solve_pyramid = solve_pyramid
    fisheyestereo.solve_pyramid = solve_pyramid
    try:  # the CLI calls through `solver.solve_pyramid` (same module object)
        import fisheyestereo.cli  # noqa: F401
    except Exception:
        pass


def uninstall() -> None:
    """Restore the reference's own solve_pyramid."""
    global _original
    if _original is None:
        return
    import fisheyestereo
    import fisheyestereo.solver as ref_solver
    ref_solver.solve_pyramid = _original
    fisheyestereo.solve_pyramid = _original
    _original = None


def calls() -> int:
    """Number of solves routed to the B200 path since import."""
    return _calls


# ---------------------------------------------------------------- pytest plugin

def pytest_configure(config):  # noqa: D401 - pytest hook
    install(os.environ.get("FSB_DROPIN_PRECISION", "fp64"))


def pytest_unconfigure(config):  # noqa: D401 - pytest hook
    out = os.environ.get("FSB_DROPIN_COUNT")
    if out:
        with open(out, "w") as f:
            f.write(str(_calls))
