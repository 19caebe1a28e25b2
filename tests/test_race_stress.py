"""Race stress of the cluster / chain kernels (the compute-sanitizer is
closed on this pool: runs under it have left GPUs needing a reset).  A build
with -DSWR_RACE_STRESS=1 delays a pseudo-random quarter of the warps by up to
~2 us at every synchronisation site of k_march (constant and time-dependent
matrix: cluster scans by st.async + mbarrier), k_march_nl (cluster barriers)
and k_march_stream (chains of CTAs with release/acquire flags).  Any missing
ordering between CTAs then shows up as a different result: the stressed
library must reproduce the normal build bitwise on shapes with multi-CTA
clusters and chains.  (Round 1's advisor found such an ordering gap in the
streaming march's halo reads; it is fixed and this test guards it.)"""
import numpy as np
import pytest

import swr_inputs as si

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def libs():
    import torch
    assert torch.cuda.is_available()
    import paper_1503_02564_b200 as pkg
    from paper_1503_02564_b200 import _build
    stressed = pkg.swr.load(_build.build_variant("race_stress", ["-DSWR_RACE_STRESS=1"]))
    return pkg, pkg.lib(), stressed


def _u0(p):
    x = p.nodes()
    return np.exp(-(x * x) / 1e-3 + 2j * x)


CASES = [
    # resident march, C5 subdomain size (M = 11, P = 256, 3-CTA cluster)
    ("march-cs3", si.Problem(a0=-0.42, b0=0.42, T=0.02, dx=1e-5, dt=1e-3, N=10, potential=si.POT_VX)),
    # time-dependent factors (per-step bulk copies), same cluster shape
    ("march-tdm", si.Problem(a0=-0.42, b0=0.42, T=0.02, dx=1e-5, dt=1e-3, N=10, potential=si.POT_VTX,
                             algorithm=si.ALG_PRECOND)),
    # nonlinear march, multi-CTA cluster with cluster-wide fixed-point stops
    ("march-nl", si.Problem(a0=-0.42, b0=0.42, T=0.01, dx=1e-5, dt=1e-3, N=10, potential=si.POT_CUBIC,
                            algorithm=si.ALG_PRECOND)),
    # streaming march, chains of co-resident CTAs
    ("march-stream", si.Problem(a0=-0.42, b0=0.42, T=0.02, dx=1e-5, dt=1e-3, N=10, potential=si.POT_VX,
                                march_form=1)),
    # streaming NL march: chain-wide fixed-point stops through published maxima
    ("march-nl-stream", si.Problem(a0=-0.42, b0=0.42, T=0.01, dx=1e-5, dt=1e-3, N=10, potential=si.POT_CUBIC,
                                   algorithm=si.ALG_PRECOND, march_form=1)),
]


@pytest.mark.parametrize("name,p", CASES, ids=[c[0] for c in CASES])
def test_stressed_kernels_bitwise(libs, name, p):
    import torch
    pkg, normal, stressed = libs
    arrays = si.inputs(p)
    arrays["u0"] = _u0(p)
    rng = np.random.default_rng(1)
    g = torch.as_tensor(rng.standard_normal(p.ng) + 1j * rng.standard_normal(p.ng), device="cuda")
    out = []
    for L in (normal, stressed, stressed):
        s = pkg.SWR(p, arrays, library=L)
        Rg, uT = s.apply_R(g, use_u0=True, want_uT=True)
        torch.cuda.synchronize()
        out.append((Rg.cpu().numpy(), uT.cpu().numpy()))
        s.close()
    for o in out[1:]:
        assert np.array_equal(o[0], out[0][0]) and np.array_equal(o[1], out[0][1]), name
