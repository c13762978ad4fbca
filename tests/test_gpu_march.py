"""The experimental i-marching colour-fused red-black kernel (LESB_SOR_MARCH=1,
solver path 3) against the golden vectors of the reference: bitwise."""

import os

import numpy as np
import pytest

import golden_inputs as gi

pytestmark = pytest.mark.gpu


@pytest.fixture()
def march():
    import paper_1504_02264_b200 as P

    os.environ["LESB_SOR_MARCH"] = "1"
    P.runtime.set_sor_path(3)
    yield P
    P.runtime.set_sor_path(0)
    os.environ.pop("LESB_SOR_MARCH", None)


@pytest.mark.parametrize("tag,dims,h", gi.SOR_CASES)
def test_march_sor_bitwise(march, tag, dims, h):
    P = march
    GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "small.npz"))
    p0, rhs = gi.sor_problem(*dims, seed=gi.seed_of(tag))
    grid = P.Grid.uniform(*dims, h)
    c = P.sor.build_uniform_coeffs(grid)
    for pol, fn in (("stored", None), ("press", P.les._pressure_halo(grid))):
        p, res = P.sor.solve_pressure(p0.copy(), rhs, c, 1.7, 9, P.Scheme.REDBLACK, 1, halo_fn=fn)
        exp = GOLD[f"{tag}/redblack/{pol}/p"]
        assert np.array_equal(p.view(np.uint32), exp.view(np.uint32)), pol
        np.testing.assert_allclose(res, GOLD[f"{tag}/redblack/{pol}/res"], rtol=1e-12, atol=0)
