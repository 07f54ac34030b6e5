"""Multi-rank host logic on CPU (gloo, world size 2): the row partition and the
collective schedule of the distributed mBCG, replayed with the
fp64 oracle's arithmetic per rank and checked against the single-process oracle.

Per iteration the library all-gathers the search directions and all-reduces
three per-column fp64 partial sums; this test runs exactly that schedule with
torch.distributed (gloo) so a wrong partition, a missing reduction or a
mis-ordered exchange shows up as a mismatch."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def row_partition(n, nranks, rank):
    # import inside: the package raises without libbbmm.so, the rule is pure Python
    from paper_1809_11165_b200 import row_partition as rp
    return rp(n, nranks, rank)


def test_partition_covers_rows_and_aligns_tiles():
    for n in (1, 127, 128, 129, 1000, 3338, 45730, 200_000, 1_000_000):
        for G in (1, 2, 3, 4, 8):
            parts = [row_partition(n, G, r) for r in range(G)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            for (a0, a1, nb), (b0, b1, _) in zip(parts, parts[1:]):
                assert a1 == b0
            for r0, r1, nb in parts:
                assert nb % 128 == 0 and r1 - r0 <= nb
                assert r0 == r1 or r0 % 128 == 0


def _worker(rank, world, port, out):
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.dataclasses.replace(synth.scaled(synth.CONFIGS["C4"], 300), k=8, t=4, p=6)
    pr = synth.make_problem(cfg, seed=0)
    n, c = cfg.n, cfg.t + 1
    r0, r1, nb = row_partition(n, world, rank)
    L, _, ku, _ = oracle.pivchol_kernel(cfg.kind, pr.X, pr.log_ls, pr.log_s, cfg.k)
    s2 = math.exp(2 * pr.log_noise)
    B = synth.random_block(n, c, seed=5).astype(np.float64)
    Lloc, Bloc = L[r0:r1], B[r0:r1]
    ch, _ = oracle.precond_setup(L, s2)

    def allreduce(x):
        t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
        dist.all_reduce(t)
        return t.numpy()

    def allgather_rows(x_loc):
        pad = np.zeros((nb, c))
        pad[: r1 - r0] = x_loc
        bufs = [torch.zeros(nb, c, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(bufs, torch.from_numpy(pad))
        return np.concatenate([b.numpy() for b in bufs])[:n]

    def precond(Rloc):
        # W = L^T R: local partial + all-reduce; S = C^-1 W; Z = (R - L S)/sigma^2
        W = allreduce(Lloc.T @ Rloc)
        S = np.linalg.solve(ch.T, np.linalg.solve(ch, W))
        return (Rloc - Lloc @ S) / s2

    U = np.zeros_like(Bloc)
    R = Bloc.copy()
    Z = precond(R)
    D = Z.copy()
    rho = allreduce((R * Z).sum(0))
    alphas = []
    for _ in range(cfg.p):
        Dfull = allgather_rows(D)
        V = oracle.kernel_matmul(cfg.kind, pr.X, pr.log_ls, pr.log_s, pr.log_noise, Dfull,
                                 rows=np.arange(r0, r1))
        dv = allreduce((D * V).sum(0))
        a = rho / dv
        alphas.append(a)
        U += a * D
        R -= a * V
        Z = precond(R)
        rz = allreduce((R * Z).sum(0))
        D = Z + (rz / rho) * D
        rho = rz
    Ufull = allgather_rows(U)
    if rank == 0:
        ro = oracle.mbcg_kernel(cfg.kind, pr.X, pr.log_ls, pr.log_s, pr.log_noise, B, cfg.p, L=L)
        out["err"] = float(np.abs(Ufull - ro["U"]).max() / np.abs(ro["U"]).max())
        out["aerr"] = float(np.abs(np.array(alphas) - ro["alpha"]).max())
    dist.barrier()
    dist.destroy_process_group()


def test_distributed_mbcg_schedule_matches_oracle():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out["err"] < 1e-10, out["err"]
    assert out["aerr"] < 1e-10, out["aerr"]
