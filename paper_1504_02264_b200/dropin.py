"""Install the CUDA path behind the reference's own operator API.

The reference (gmcf_mini, pure Python) has no plugin registry: its callers
resolve the hot-path functions through module globals at call time
(``les_main`` calls ``step``, les.py:460; ``cli`` calls ``les.step``,
cli.py:208, and ``sor.solve_pressure``, cli.py:234 and 253; ``press`` calls
``sor.solve_pressure``, les.py:376).  ``install()`` rebinds those globals to
this package's functions, which take the reference's own FlowState,
WindProfile, Scheme and halo_fn objects; ``uninstall()``
restores the originals.

    import gmcf_mini
    import paper_1504_02264_b200 as b200
    b200.install()          # every les.step / solve_pressure now runs on the GPU
"""

from __future__ import annotations

import importlib

from . import cli as _cli
from . import les as _les
from . import sor as _sor

LES_FUNCS = ("step", "velnw", "bondv1", "velfg_merged", "velfg_twopass", "feedbf", "les_viscosity",
             "strain_magnitude", "adam", "divergence", "press", "les_main")
CLI_FUNCS = ("les_main", "run_boundary_audit")  # cli.py:23 binds les_main at import
# cli.main dispatches through the _RUNNERS table built at import (cli.py:323-328):
# mode -> (module, function) of the device implementation
CLI_RUNNERS = {"boundary-audit": (_les, "run_boundary_audit"), "les-standalone": (_cli, "run_les_standalone"),
               "sor-bench": (_cli, "run_sor_bench")}
SOR_FUNCS = ("solve_pressure", "redblack_iteration", "twinned_sweep")
# gmcf_mini/__init__.py re-exports les_main and the solver entry points
# (``from gmcf_mini import solve_pressure`` binds the package attribute)
PKG_LES_FUNCS = ("les_main",)
PKG_SOR_FUNCS = SOR_FUNCS

_saved: dict = {}


def install(les_module=None, sor_module=None) -> None:
    """Rebind gmcf_mini.les / gmcf_mini.sor hot-path functions to the CUDA
    implementations (idempotent)."""
    lm = les_module or importlib.import_module("gmcf_mini.les")
    sm = sor_module or importlib.import_module("gmcf_mini.sor")
    mods = [(lm, LES_FUNCS, _les), (sm, SOR_FUNCS, _sor)]
    if les_module is None:
        try:
            mods.append((importlib.import_module("gmcf_mini.cli"), CLI_FUNCS, _les))
        except ImportError:
            pass
        try:
            pkg = importlib.import_module("gmcf_mini")
            mods.append((pkg, PKG_LES_FUNCS, _les))
            mods.append((pkg, PKG_SOR_FUNCS, _sor))
        except ImportError:
            pass
    for mod, names, impl in mods:
        for n in names:
            if not hasattr(mod, n):
                continue
            key = (mod.__name__, n)
            if key not in _saved:
                _saved[key] = (mod, getattr(mod, n))
            setattr(mod, n, getattr(impl, n))
        runners = getattr(mod, "_RUNNERS", None) if names is CLI_FUNCS else None
        if isinstance(runners, dict):
            for mode, (rmod, fn) in CLI_RUNNERS.items():
                if mode in runners:
                    key = (mod.__name__, "_RUNNERS:" + mode)
                    if key not in _saved:
                        _saved[key] = (runners, runners[mode])
                    runners[mode] = getattr(rmod, fn)


def uninstall() -> None:
    """Restore the reference implementations."""
    for (_modname, n), (mod, fn) in list(_saved.items()):
        if n.startswith("_RUNNERS:"):
            mod[n[len("_RUNNERS:"):]] = fn
        else:
            setattr(mod, n, fn)
    _saved.clear()


def installed() -> bool:
    return bool(_saved)
