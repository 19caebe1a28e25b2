"""Multi-rank protocol on CPU (gloo, world_size 2 and 3): the partition and
slot ownership of libswr (swr_partition, swr_owned_slots -- host functions of
the library, no GPU needed) with the exchange rules the library applies
(SURVEY 8(e)): every rank keeps only its own interface slots, the outputs of
its subdomains that land in a neighbour's slot travel as cut traces by
point-to-point send/recv, dot products are per-subdomain partials summed
over ranks (disjoint columns) and reduced in subdomain order, u(T) nodes
shared across a cut get half of each copy.  One sweep R(g), its dot
products and u(T) reproduce the single-process results bitwise.  The
per-subdomain marches are the oracle's; libswr's device code path for the
same protocol runs in tests/test_multirank.py (logical ranks on one GPU)."""
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


def test_owned_slots_tile_the_interface_vector():
    from paper_1503_02564_b200.swr import owned_slots, partition
    for N in (2, 3, 10, 97, 500):
        for W in (1, 2, 3, 4, 8):
            if W > N:
                continue
            prev = -1
            for r in range(W):
                lo, hi = owned_slots(N, W, r)
                jl, jh = partition(N, W, r)
                assert lo == prev + 1 and lo == (0 if jl == 1 else 2 * jl - 3)
                assert hi == (2 * N - 3 if jh == N else 2 * jh - 2)
                prev = hi
            assert prev == 2 * N - 3


def _inputs(p):
    d = si.inputs(p)
    x = p.nodes()
    d["u0"] = np.exp(-(x + 1.0) ** 2 + 3j * x)
    return d


def _rank_step(rank, world, o, p, g, send, recv, allreduce):
    """One sweep R(g) + the dot <R(g), R(g)> + u(T) under the library's
    protocol on one rank; send/recv/allreduce are the transport."""
    from paper_1503_02564_b200.swr import owned_slots, partition
    NT, N, m = p.NT, p.N, p.Nx // p.N
    jlo, jhi = partition(N, world, rank)
    slo, shi = owned_slots(N, world, rank)
    gl = g[slo * NT:(shi + 1) * NT]                       # this rank's slots only
    Rg = np.zeros_like(gl)
    halo = {}
    loc = {}

    def put(slot, val):                                   # local slot or cut trace
        if slo <= slot <= shi:
            Rg[(slot - slo) * NT:(slot - slo + 1) * NT] = val
        else:
            halo["L" if slot < slo else "R"] = val

    for j in range(jlo, jhi + 1):
        lin = gl[(2 * j - 3 - slo) * NT:(2 * j - 2 - slo) * NT] if j >= 2 else None
        rin = gl[(2 * j - 2 - slo) * NT:(2 * j - 1 - slo) * NT] if j <= N - 1 else None
        st, ol, orr, ul, _ = o.march(j, lin, rin, use_u0=True)
        if j >= 2:
            put(2 * j - 4, ol)
        if j <= N - 1:
            put(2 * j - 1, orr)
        loc[j] = ul
    # cut traces: to the left neighbour its last slot, to the right its first
    # (posted sends, then the receives: the ncclGroupStart/End pattern)
    reqs = []
    if rank > 0:
        reqs.append(send(halo["L"], rank - 1))
    if rank < world - 1:
        reqs.append(send(halo["R"], rank + 1))
    if rank > 0:
        Rg[:NT] = recv(rank - 1)
    if rank < world - 1:
        Rg[-NT:] = recv(rank + 1)
    for q in reqs:
        q.wait()
    # dot: per-subdomain partials (the subdomain's own slots), summed over ranks, then in order
    part = np.zeros(N, np.complex128)
    for j in range(jlo, jhi + 1):
        a, b = (2 * j - 3 if j >= 2 else 0), (2 * j - 2 if j <= N - 1 else 2 * N - 3)
        v = Rg[(a - slo) * NT:(b - slo + 1) * NT]
        part[j - 1] = np.vdot(v, v)
    part = allreduce(part)
    dot = complex(0.0)
    for j in range(N):
        dot += part[j]
    # u(T): own nodes, half of each copy at a node shared with a neighbour rank
    uT = np.zeros(p.Nx + 1, np.complex128)
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
    uT = allreduce(uT)
    return Rg, slo, shi, dot, uT


def _worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist
    from oracle import oracle
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    p = si.Problem(**PROBLEM)
    o = oracle.Oracle(p, _inputs(p))
    rng = np.random.default_rng(3)
    g = rng.standard_normal(o.ng) + 1j * rng.standard_normal(o.ng)

    def send(v, dst):
        return dist.isend(torch.from_numpy(np.ascontiguousarray(v).view(np.float64).copy()), dst)

    def recv(src):
        t = torch.zeros(2 * p.NT, dtype=torch.float64)
        dist.recv(t, src)
        return t.numpy().view(np.complex128)

    def allreduce(a):
        t = torch.from_numpy(np.ascontiguousarray(a).view(np.float64).copy())
        dist.all_reduce(t)
        return t.numpy().view(np.complex128)

    Rg, slo, shi, dot, uT = _rank_step(rank, world, o, p, g, send, recv, allreduce)
    np.savez(os.path.join(outdir, f"r{rank}.npz"), Rg=Rg, slo=slo, shi=shi, dot=dot, uT=uT, g=g)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ranks_match_single_process(oracle_mod, tmp_path, world):
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    p = si.Problem(**PROBLEM)
    o = oracle_mod.Oracle(p, _inputs(p))
    res = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    g = res[0]["g"]
    ident = lambda a: a  # noqa: E731  (one rank: no transport)
    Rg1, _, _, dot1, uT1 = _rank_step(0, 1, o, p, g, None, None, ident)
    assert np.array_equal(Rg1, o.apply_R(g, use_u0=True))
    NT = p.NT
    for r in res:
        assert np.array_equal(r["Rg"], Rg1[int(r["slo"]) * NT:(int(r["shi"]) + 1) * NT])
        assert complex(r["dot"]) == dot1
        assert np.array_equal(r["uT"], uT1)
