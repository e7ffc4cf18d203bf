"""Multi-process tests of the sequence-parallel scan (paper_2312_06635_b200/parallel.py).

CPU: world_size 2 and 4 over gloo (127.0.0.1); the local operators are the fp64 oracle (test infrastructure),
so these tests check the scan algebra and the send/recv pattern exactly (1e-11).
GPU: the same algebra with the CUDA operators on virtual ranks (segments processed in order in one process),
against the oracle on the whole sequence.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2312_06635_b200 import parallel as P

B, H, T, K, V = 1, 2, 96, 4, 6


def _np(t):
    return None if t is None else t.detach().double().cpu().numpy()


def oracle_ops():
    def summary(k, v, g):
        _, fs = oracle.fwd(np.zeros(_np(k).shape), _np(k), _np(v), _np(g))
        return torch.from_numpy(fs), torch.from_numpy(_np(g).sum(axis=2))

    def dsummary(q, do, g):
        Vd = do.shape[-1]
        z = np.zeros(_np(q).shape)
        return torch.from_numpy(oracle.bwd(_np(q), z, np.zeros(z.shape[:-1] + (Vd,)), _np(g), _np(do))[4])

    def combine(h, d, s):
        return torch.exp(d)[..., None] * h + s

    def fwd(q, k, v, g, h0):
        o, fs = oracle.fwd(_np(q), _np(k), _np(v), _np(g), h0=_np(h0))
        return torch.from_numpy(o), torch.from_numpy(fs)

    def bwd(q, k, v, g, do, h0, dfin):
        return tuple(torch.from_numpy(x) for x in oracle.bwd(_np(q), _np(k), _np(v), _np(g), _np(do), h0=_np(h0),
                                                            d_final=_np(dfin)))

    return P.LocalOps(summary, dsummary, combine, fwd, bwd)


def full_problem():
    p = synth.problem(B, H, T, K, V, seed=3, gate="strong", dtype=torch.float64)
    p["h0"] = synth.state(B, H, K, V, 1).double()
    p["dfin"] = synth.state(B, H, K, V, 2).double()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = full_problem()
    seg = T // world
    sl = slice(rank * seg, (rank + 1) * seg)
    q, k, v, g, do = (p[n][:, :, sl].contiguous() for n in ("q", "k", "v", "g", "do"))
    ops = oracle_ops()
    o, fs, ctx = P.sp_forward(q, k, v, g, ops, initial_state=p["h0"] if rank == 0 else None)
    grads = P.sp_backward(q, k, v, g, do, ctx, ops, d_final_state=p["dfin"] if rank == world - 1 else None)
    torch.save({"o": o, "fs": fs, "grads": grads}, os.path.join(out, f"r{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world", [2, 4])
def test_sp_scan_gloo(tmp_path, world):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    res = [torch.load(os.path.join(tmp_path, f"r{r}.pt")) for r in range(world)]
    p = full_problem()
    f = {n: _np(p[n]) for n in ("q", "k", "v", "g", "do", "h0", "dfin")}
    ro, rfs = oracle.fwd(f["q"], f["k"], f["v"], f["g"], h0=f["h0"])
    rdq, rdk, rdv, rdg, rdh0 = oracle.bwd(f["q"], f["k"], f["v"], f["g"], f["do"], h0=f["h0"], d_final=f["dfin"])
    o = np.concatenate([_np(r["o"]) for r in res], axis=2)
    np.testing.assert_allclose(o, ro, rtol=1e-11, atol=1e-11)
    np.testing.assert_allclose(_np(res[-1]["fs"]), rfs, rtol=1e-11, atol=1e-11)
    for i, ref in enumerate((rdq, rdk, rdv, rdg)):
        got = np.concatenate([_np(r["grads"][i]) for r in res], axis=2)
        np.testing.assert_allclose(got, ref, rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(_np(res[0]["grads"][4]), rdh0, rtol=1e-10, atol=1e-10)


def test_shard_bh_covers_batch():
    for Bt in (1, 5, 16):
        for w in (1, 2, 3, 8):
            cov = []
            for r in range(w):
                b0, b1 = P.shard_bh(Bt, r, w)
                cov.extend(range(b0, b1))
            assert cov == list(range(Bt))


@pytest.mark.gpu
@pytest.mark.parametrize("R", [2, 4])
def test_sp_virtual_ranks_cuda(R):
    """The CUDA operators composed through the same scan on R virtual ranks == single-pass oracle."""
    from tests.helpers import nerr_slices
    Bc, Hc, Tc, Kc, Vc = 1, 2, 512, 128, 256
    p = synth.problem(Bc, Hc, Tc, Kc, Vc, seed=5)
    pc = {n: t.cuda() for n, t in p.items()}
    ops = P.cuda_ops()
    seg = Tc // R
    parts = [{n: pc[n][:, :, r * seg:(r + 1) * seg].contiguous() for n in pc} for r in range(R)]
    Hs, Ds = [torch.zeros(Bc, Hc, Kc, Vc, device="cuda")], []
    for r in range(R):
        S, D = ops.state_summary(parts[r]["k"], parts[r]["v"], parts[r]["g"])
        Ds.append(D)
        Hs.append(ops.state_combine(Hs[-1], D, S))
    outs = [ops.chunk_fwd(parts[r]["q"], parts[r]["k"], parts[r]["v"], parts[r]["g"], Hs[r])[0] for r in range(R)]
    dF = [None] * R
    dF[R - 1] = torch.zeros(Bc, Hc, Kc, Vc, device="cuda")
    for r in range(R - 1, 0, -1):
        dh = ops.dstate_summary(parts[r]["q"], parts[r]["do"], parts[r]["g"])
        dF[r - 1] = ops.state_combine(dF[r], Ds[r], dh)
    grads = [ops.chunk_bwd(parts[r]["q"], parts[r]["k"], parts[r]["v"], parts[r]["g"], parts[r]["do"], Hs[r], dF[r])
             for r in range(R)]
    torch.cuda.synchronize()
    f = {n: p[n].double().numpy() for n in p}
    ro, _ = oracle.fwd(f["q"], f["k"], f["v"], f["g"])
    rg = oracle.bwd(f["q"], f["k"], f["v"], f["g"], f["do"])
    o = torch.cat(outs, 2).float().cpu().numpy()
    assert nerr_slices(o, ro) < 2e-2
    for i in range(3):
        got = torch.cat([gr[i] for gr in grads], 2).float().cpu().numpy()
        assert nerr_slices(got, rg[i]) < 2e-2, i
