"""Multi-rank path on CPU (gloo, world_size 2): the subdomain partition of
libswr (swr_partition) and the assembly rules the library applies with
ncclAllReduce — every rank fills only its own subdomains' outputs (disjoint
supports), interface nodes shared across a rank cut get half of each copy —
reproduce the single-process results bitwise.  The per-subdomain marches are
the oracle's; the assembly/exchange logic is what is under test."""
import os
import socket

import numpy as np
import pytest

import swr_inputs as si


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_partition_covers_contiguously():
    from paper_1503_02564_b200.swr import partition
    for N in (1, 2, 3, 10, 97, 500, 1000):
        for W in (1, 2, 3, 4, 8):
            if W > N:
                continue
            ranges = [partition(N, W, r) for r in range(W)]
            assert ranges[0][0] == 1 and ranges[-1][1] == N
            for (a, b), (c, d) in zip(ranges, ranges[1:]):
                assert c == b + 1
            sizes = [b - a + 1 for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 1


PROBLEM = dict(a0=-7.0, b0=7.0, T=0.06, dx=0.1, dt=0.01, N=7, potential=si.POT_VX, transmission=si.TC_S02,
               vx_kind="-x2")


def _inputs(p):
    d = si.inputs(p)
    x = p.nodes()
    d["u0"] = np.exp(-(x + 1.0) ** 2 + 3j * x)
    return d


def _worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist
    from oracle import oracle
    from paper_1503_02564_b200.swr import partition
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    p = si.Problem(**PROBLEM)
    o = oracle.Oracle(p, _inputs(p))
    NT, N, m, Nj = p.NT, p.N, p.Nx // p.N, p.Nj
    jlo, jhi = partition(N, world, rank)
    rng = np.random.default_rng(3)
    g = rng.standard_normal(o.ng) + 1j * rng.standard_normal(o.ng)
    Rg = np.zeros(o.ng, np.complex128)
    X = np.zeros((N, 4, NT), np.complex128)
    uT = np.zeros(p.Nx + 1, np.complex128)
    e = np.zeros(NT, np.complex128)
    e[0] = 1
    loc = {}
    for j in range(jlo, jhi + 1):
        lin = g[(2 * j - 3) * NT:(2 * j - 2) * NT] if j >= 2 else None
        rin = g[(2 * j - 2) * NT:(2 * j - 1) * NT] if j <= N - 1 else None
        st, ol, orr, ul, _ = o.march(j, lin, rin, use_u0=True)
        if j >= 2:
            Rg[(2 * j - 4) * NT:(2 * j - 3) * NT] = ol
        if j <= N - 1:
            Rg[(2 * j - 1) * NT:(2 * j) * NT] = orr
        loc[j] = ul
        if j >= 2:
            _, a, b, _, _ = o.march(j, e, None, use_u0=False)
            X[j - 1, 0] = a
            if j <= N - 1:
                X[j - 1, 2] = b
        if j <= N - 1:
            _, a, b, _, _ = o.march(j, None, e, use_u0=False)
            if j >= 2:
                X[j - 1, 1] = a
            X[j - 1, 3] = b
    # u(T) gather rule of k_gather_uT (multi-GPU form)
    for i in range(p.Nx + 1):
        j0 = (N - 1) if i == p.Nx else i // m
        k = i - j0 * m
        own = jlo <= j0 + 1 <= jhi
        v = loc[j0 + 1][k] if own else 0
        if k == 0 and j0 > 0:
            ownl = jlo <= j0 <= jhi
            w = loc[j0][m] if ownl else 0
            if own and ownl:
                v = (w + v) / 2
            elif own:
                v = v / 2
            elif ownl:
                v = w / 2
        uT[i] = v
    for arr in (Rg, X, uT):
        t = torch.from_numpy(arr.view(np.float64).reshape(-1))
        dist.all_reduce(t)
        arr.view(np.float64).reshape(-1)[:] = t.numpy()
    if rank == 0:
        np.savez(os.path.join(outdir, "res.npz"), Rg=Rg, X=X, uT=uT, g=g)
    dist.destroy_process_group()


def test_two_rank_assembly_matches_single_process(oracle_mod, tmp_path):
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    r = np.load(tmp_path / "res.npz")
    p = si.Problem(**PROBLEM)
    o = oracle_mod.Oracle(p, _inputs(p))
    assert np.array_equal(r["Rg"], o.apply_R(r["g"], use_u0=True))
    assert np.array_equal(r["X"], o.build_L())
    # u(T) of the same sweep on one process (mean of the two copies)
    m = p.Nx // p.N
    s = np.zeros(p.Nx + 1, np.complex128)
    c = np.zeros(p.Nx + 1)
    g = r["g"]
    NT = p.NT
    for j in range(1, p.N + 1):
        lin = g[(2 * j - 3) * NT:(2 * j - 2) * NT] if j >= 2 else None
        rin = g[(2 * j - 2) * NT:(2 * j - 1) * NT] if j <= p.N - 1 else None
        ul = o.march(j, lin, rin, use_u0=True)[3]
        s[(j - 1) * m:(j - 1) * m + p.Nj] += ul
        c[(j - 1) * m:(j - 1) * m + p.Nj] += 1
    assert np.array_equal(r["uT"], s / c)
