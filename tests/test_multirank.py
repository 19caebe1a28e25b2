"""libswr's real multi-rank code path (owner-computes slots, cut-trace
exchange, exchanged per-subdomain partial sums, u(T) reduction) on one GPU:
G = 2, 3 and 4 logical ranks run as host threads of this process, each with
its own handle and stream, joined by the library's loopback communicator
(device copies standing in for NCCL; swr_loopback_id, test infrastructure).
The iterates must be bitwise those of one rank (the order-fixed
reductions make the sharding invisible): iteration counts, every residual
estimate, each rank's slots of g, u(T) on rank 0, the NL fixed-point maxima.
"""
import threading

import numpy as np
import pytest

import swr_inputs as si

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1503_02564_b200 as pkg
    pkg.lib()
    return pkg


def _run_ranks(pkg, p, arrays, G, timeout=240):
    import torch
    lid = pkg.swr.loopback_id(G)
    out = [None] * G
    errors = []

    def run(r):
        try:
            torch.cuda.set_device(0)
            stream = torch.cuda.Stream()
            s = pkg.SWR(p, arrays, stream=stream, rank=r, world=G, nccl_id=lid)
            s.build()
            st, uT, rep = s.solve()
            g = s.get_g().cpu().numpy()
            out[r] = dict(st=st, uT=uT, rep=rep, g=g, s_lo=s.s_lo, s_hi=s.s_hi)
            s.close()
        except Exception as e:   # noqa: BLE001  (reported below)
            errors.append((r, repr(e)))

    threads = [threading.Thread(target=run, args=(r,), daemon=True) for r in range(G)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout)
    assert not any(t.is_alive() for t in threads), "a logical rank hung"
    assert not errors, errors
    return out


CASES = [
    ("new-gmres", si.config("C1", transmission=si.TC_S02, potential=si.POT_VX, N=8)),
    ("new-bicgstab", si.config("C1", transmission=si.TC_S02, potential=si.POT_VX, N=8, krylov=si.KRY_BICGSTAB)),
    ("new-robin-direct", si.config("C1", transmission=si.TC_ROBIN, potential=si.POT_VX, N=5, robin_p=19.0,
                                   toeplitz_form=1)),
    ("classical-fp", si.config("C1", transmission=si.TC_S02, potential=si.POT_VX, N=8, algorithm=si.ALG_CLASSICAL,
                               krylov=si.KRY_FIXED_POINT)),
    ("precond-vtx", si.config("C1", transmission=si.TC_S02, potential=si.POT_VTX, N=8, algorithm=si.ALG_PRECOND)),
    ("precond-nl-exact", si.config("C1", transmission=si.TC_S02, potential=si.POT_CUBIC, N=8,
                                   algorithm=si.ALG_PRECOND, krylov=si.KRY_FIXED_POINT, u0_kind="soliton",
                                   pinv_exact=1)),
    ("mid-N42-stream", si.Problem(dx=1e-3, dt=5e-3, N=42, potential=si.POT_VX, march_form=1)),
    ("precond-nl-stream", si.config("C1", transmission=si.TC_S02, potential=si.POT_CUBIC, N=8,
                                    algorithm=si.ALG_PRECOND, krylov=si.KRY_FIXED_POINT, u0_kind="soliton",
                                    pinv_exact=1, march_form=1)),
]


@pytest.mark.timeout(600)
@pytest.mark.parametrize("G", [2, 3, 4])
@pytest.mark.parametrize("name,p", CASES, ids=[c[0] for c in CASES])
def test_logical_ranks_bitwise_one_rank(gpu, name, p, G):
    arrays = si.inputs(p)
    s1 = gpu.SWR(p, arrays)
    s1.build()
    st1, u1, r1 = s1.solve()
    g1 = s1.get_g().cpu().numpy()
    s1.close()
    assert st1 == 0
    out = _run_ranks(gpu, p, arrays, G)
    NT = p.NT
    covered = 0
    for r, o in enumerate(out):
        assert o["st"] == 0, (r, o["st"])
        assert o["rep"]["iterations"] == r1["iterations"], (r, o["rep"]["iterations"], r1["iterations"])
        assert o["rep"]["inner_iterations"] == r1["inner_iterations"]
        assert o["rep"]["fp_max"] == r1["fp_max"]
        assert np.array_equal(o["rep"]["history"], r1["history"]), r
        assert np.array_equal(o["g"], g1[o["s_lo"] * NT:(o["s_hi"] + 1) * NT]), r
        covered += o["s_hi"] - o["s_lo"] + 1
    assert covered == 2 * p.N - 2
    assert np.array_equal(out[0]["uT"], u1)
