"""The NCCL path of libswr on real GPUs (one process per GPU, torchrun-style
ranks over 127.0.0.1): a 2-rank solve of the NEW algorithm must reproduce
the one-GPU iterates bitwise (iteration count, residual history, u(T) on
rank 0, each rank's slots of g).  Skipped on machines with fewer than two
GPUs (this pool's boxes have one; the same multi-rank code path runs with
logical ranks in tests/test_multirank.py)."""
import os
import socket

import numpy as np
import pytest

import swr_inputs as si

pytestmark = pytest.mark.gpu

P = dict(name="C1", transmission=si.TC_S02, potential=si.POT_VX, N=8)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist
    import paper_1503_02564_b200 as pkg
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    kw = dict(P)
    p = si.config(kw.pop("name"), **kw)
    obj = [pkg.swr.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    s = pkg.SWR(p, si.inputs(p), device=rank, rank=rank, world=world, nccl_id=obj[0])
    s.build()
    st, uT, rep = s.solve()
    g = s.get_g().cpu().numpy()
    np.savez(os.path.join(outdir, f"r{rank}.npz"), st=st, uT=uT, hist=rep["history"], it=rep["iterations"], g=g,
             s_lo=s.s_lo, s_hi=s.s_hi, comm=rep["t_comm_ms"])
    s.close()
    dist.destroy_process_group()


def test_two_gpus_bitwise_one_gpu(tmp_path):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    import torch.multiprocessing as mp
    import paper_1503_02564_b200 as pkg
    kw = dict(P)
    p = si.config(kw.pop("name"), **kw)
    s1 = pkg.SWR(p, si.inputs(p))
    s1.build()
    st1, u1, r1 = s1.solve()
    g1 = s1.get_g().cpu().numpy()
    s1.close()
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        o = np.load(tmp_path / f"r{r}.npz")
        assert int(o["st"]) == 0 and int(o["it"]) == r1["iterations"]
        assert np.array_equal(o["hist"], r1["history"])
        assert np.array_equal(o["g"], g1[int(o["s_lo"]) * p.NT:(int(o["s_hi"]) + 1) * p.NT])
        assert float(o["comm"]) > 0.0
        if r == 0:
            assert np.array_equal(o["uT"], u1)
