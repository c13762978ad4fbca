"""The drop-in hook rebinds exactly the reference's hot-path functions and
restores them (CPU only: no compute calls).  Needs the reference importable,
which it is in the build container; skipped elsewhere (the GPU box)."""

import os
import sys

import pytest

REF = "/root/reference/pkg/src"


@pytest.fixture()
def ref():
    if os.path.isdir(REF) and REF not in sys.path:
        sys.path.append(REF)
    les = pytest.importorskip("gmcf_mini.les")
    sor = pytest.importorskip("gmcf_mini.sor")
    return les, sor


def test_install_rebinds_and_restores(ref):
    les, sor = ref
    import paper_1504_02264_b200 as P

    orig = {n: getattr(les, n) for n in P.dropin.LES_FUNCS}
    orig.update({n: getattr(sor, n) for n in P.dropin.SOR_FUNCS})
    P.install()
    try:
        assert P.installed()
        for n in P.dropin.LES_FUNCS:
            assert getattr(les, n) is getattr(P.les, n), n
        for n in P.dropin.SOR_FUNCS:
            assert getattr(sor, n) is getattr(P.sor, n), n
        P.install()  # idempotent: originals stay recorded
    finally:
        P.uninstall()
    for n, fn in orig.items():
        mod = les if n in P.dropin.LES_FUNCS else sor
        assert getattr(mod, n) is fn, n
    assert not P.installed()


def test_reference_scheme_members_accepted(ref):
    """Scheme is compared by identity in the reference (sor.py:268, 273); the
    drop-in accepts the reference's own members as well as its own (the
    package may have been imported before gmcf_mini was importable)."""
    les, sor = ref
    from paper_1504_02264_b200 import les as L
    from paper_1504_02264_b200 import reftypes

    assert reftypes.is_redblack(sor.Scheme.REDBLACK) and not reftypes.is_redblack(sor.Scheme.TWINNED)
    assert reftypes.is_twinned(sor.Scheme.TWINNED)
    assert reftypes.is_redblack(reftypes.Scheme.REDBLACK)
    assert L._scheme_code(sor.Scheme.REDBLACK) == 0 and L._scheme_code(sor.Scheme.TWINNED) == 1
    with pytest.raises(ValueError):
        L._scheme_code("redblack")


def test_reference_pressure_halo_maps_to_press_policy(ref):
    les, sor = ref
    from paper_1504_02264_b200 import _native as N
    from paper_1504_02264_b200 import sor as S

    grid = sor.Grid.uniform(4, 5, 3, 1.0)
    assert S.halo_policy(les._pressure_halo(grid), (6, 7, 5)) == N.LESB_HALO_PRESS
    assert S.halo_policy(None, (6, 7, 5)) == N.LESB_HALO_STORED
    with pytest.raises(NotImplementedError):
        S.halo_policy(lambda p: None, (6, 7, 5))
    with pytest.raises(ValueError):
        S.halo_policy(S.PressureHalo(grid), (6, 8, 5))


def test_install_rebinds_cli_runners(ref):
    """cli.main dispatches through _RUNNERS (cli.py:323-328): install() swaps
    the boundary-audit, les-standalone and sor-bench runners for the GPU ones
    and uninstall() restores them; coupled keeps the reference's runner
    (which reaches the device through the rebound les_main)."""
    cli = pytest.importorskip("gmcf_mini.cli")
    import paper_1504_02264_b200 as P

    orig_runners = dict(cli._RUNNERS)
    orig_runner = cli._RUNNERS["boundary-audit"]
    orig_fn = cli.run_boundary_audit
    orig_main = cli.les_main
    P.install()
    try:
        assert cli._RUNNERS["boundary-audit"] is P.les.run_boundary_audit
        assert cli.run_boundary_audit is P.les.run_boundary_audit
        assert cli.les_main is P.les.les_main
        assert cli._RUNNERS["coupled"] is cli.run_coupled
        assert cli._RUNNERS["les-standalone"] is P.cli.run_les_standalone
        assert cli._RUNNERS["sor-bench"] is P.cli.run_sor_bench
    finally:
        P.uninstall()
    assert cli._RUNNERS == orig_runners
    assert cli._RUNNERS["boundary-audit"] is orig_runner
    assert cli.run_boundary_audit is orig_fn
    assert cli.les_main is orig_main


def test_resolve_accepts_reference_flowstate(ref):
    """the reference FlowState is an unhashable dataclass;
    the compat path caches its device twin by id and evicts it with the
    caller's object (no compute: FlowState construction does not touch the
    device)."""
    les, sor = ref
    import gc

    from paper_1504_02264_b200 import les as L

    st = les.FlowState.create(sor.Grid.uniform(4, 3, 2, 2.0), dt=0.5)
    with pytest.raises(TypeError):
        hash(st)
    ds, target = L._resolve(st)
    assert target is st and isinstance(ds, L.FlowState)
    assert ds._host["u"] is st.u
    ds2, t2 = L._resolve(st)
    assert ds2 is ds  # cached: one device domain per caller state
    key = id(st)
    assert key in L._compat
    del st, target, t2
    gc.collect()
    assert key not in L._compat
