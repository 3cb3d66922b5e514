"""SUMMA distributed layer: host-side logic on CPU (gloo, world sizes 2/4) and
a single-process loopback; the GPU loopback with the real kernels is -m gpu."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1605_01078_b200 import summa as SU


def dense(m, n, k, seed):
    g = torch.Generator().manual_seed(seed)
    A = torch.rand(m, k, dtype=torch.float64, generator=g) * 2 - 1
    B = torch.rand(k, n, dtype=torch.float64, generator=g) * 2 - 1
    C = torch.rand(m, n, dtype=torch.float64, generator=g) * 2 - 1
    return A, B, C


def matmul_update(alpha, a, b, c):
    c.add_(alpha * (a @ b))


def test_grids_and_layout():
    assert SU.grid_for(1) == (1, 1)
    assert SU.grid_for(2) == (1, 2)
    assert SU.grid_for(4) == (2, 2)
    assert SU.grid_for(8) == (2, 4)
    L = SU.make_layout(64, 96, 48, 8, b=4)
    assert (L.pr, L.pc, L.m_l, L.n_l, L.k_c, L.k_r, L.panels) == (2, 4, 32, 24, 12, 24, 12)
    assert L.a_owner_col(5) == (1, 8)   # k columns 20..23 live on process column 1
    assert L.b_owner_row(7) == (1, 4)   # k rows 28..31 live on process row 1
    # panels straddling owner boundaries are assembled from per-owner pieces
    L2 = SU.make_layout(64, 96, 48, 8, b=24)
    assert L2.a_pieces(1) == [(2, 0, 12, 0), (3, 0, 12, 12)]
    assert L2.b_pieces(1) == [(1, 0, 24, 0)]
    assert SU.make_layout(64, 96, 48, 8, b=48).b_pieces(0) == [(0, 0, 24, 0), (1, 0, 24, 24)]
    assert SU.make_layout(65536, 65536, 65536, 8).b == 8192
    assert SU.make_layout(32768, 65536, 16384, 8).b == 8192
    with pytest.raises(ValueError):
        SU.make_layout(64, 96, 48, 8, b=5)
    with pytest.raises(ValueError):
        SU.make_layout(63, 96, 48, 8)


@pytest.mark.parametrize("P,b", [(1, 4), (2, 4), (4, 4), (8, 4), (2, 64), (4, 64), (8, 32),
                                 (8, 64)])
def test_loopback_schedule_matches_dense(P, b):
    m, n, k = 48, 40, 64
    A, B, C = dense(m, n, k, 7)
    want = C + 0.5 * (A @ B)
    L = SU.make_layout(m, n, k, P, b=b)
    blocks = [SU.local_blocks(L, r, A, B, C) for r in range(P)]
    Cb = [c.clone() for _, _, c in blocks]
    SU.summa_loopback(L, [a for a, _, _ in blocks], [b for _, b, _ in blocks], Cb, alpha=0.5,
                      local_gemm=matmul_update)
    for r in range(P):
        _, _, wc = SU.local_blocks(L, r, A, B, want)
        assert torch.allclose(Cb[r], wc, rtol=0, atol=1e-12)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, m, n, k, b, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A, B, C = dense(m, n, k, 11)
        L = SU.make_layout(m, n, k, world, b=b)
        comm = SU.TorchComm(L)
        a, bb, c = SU.local_blocks(L, rank, A, B, C)
        c = c.clone()
        panels = SU.summa(L, comm, a.contiguous(), bb.contiguous(), c, alpha=-1.0,
                          local_gemm=matmul_update)
        want = C - A @ B
        _, _, wc = SU.local_blocks(L, rank, A, B, want)
        q.put((rank, panels, float((c - wc).abs().max())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,b", [(2, 8), (4, 4), (4, 16), (2, 64), (4, 64), (4, 32)])
def test_summa_gloo_matches_dense(world, b):
    m, n, k = 32, 48, 64
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, n, k, b, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(world))
    assert [r for r, _, _ in res] == list(range(world))
    for _, panels, err in res:
        assert panels == k // b
        assert err < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("P,variant,level,b", [(2, "abc", 1, 256), (4, "abc", 2, 256),
                                               (8, "c", 2, 256), (8, "naive", 2, 2048)])
def test_loopback_on_gpu_with_strassen_kernels(cuda, P, variant, level, b):
    """Full SUMMA data path with the real sm_100a kernels (virtual ranks, one GPU)."""
    m, n, k = 1024, 2048, 2048
    A, B, C = (x.to(cuda) for x in dense(m, n, k, 3))
    L = SU.make_layout(m, n, k, P, b=b)  # b = 2048: panels straddle A and B owners
    blocks = [SU.local_blocks(L, r, A, B, C) for r in range(P)]
    Cb = [c.t().contiguous().t() for _, _, c in blocks]  # column-major C blocks
    SU.summa_loopback(L, [a for a, _, _ in blocks], [b for _, b, _ in blocks], Cb,
                      variant=variant, level=level)
    torch.cuda.synchronize()
    want = C + A @ B
    an, bn = torch.linalg.norm(A).item(), torch.linalg.norm(B).item()
    for r in range(P):
        _, _, wc = SU.local_blocks(L, r, A, B, want)
        nw = (torch.linalg.norm(Cb[r] - wc) / (an * bn)).item()
        assert nw <= (1e-12 if level == 1 else 5e-12), (r, nw)


@pytest.mark.gpu
@pytest.mark.parametrize("N,P,variant,level", [(16384, 8, "abc", 2), (16384, 4, "naive", 2)])
def test_config5_loopback_counter_rng_sampled_tiles(cuda, N, P, variant, level):
    """BASELINE config 5's protocol at a reduced size (tools/cfg5_loopback.py runs the full
    65536^3, profiles/r01_cfg5_loopback.log): operands from the counter-based RNG, SUMMA
    over P virtual ranks with local Strassen updates, sampled 256 x 256 tiles against the
    oracle regenerated from the same counters, and a whole-matrix Freivalds check."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "tools"))
    import cfg5_loopback
    res = cfg5_loopback.run(N, P, variant, level)
    assert res["pass"], res


# ------------------------------------------------------------ peer-memory SUMMA
def test_k_pieces_cover_k_at_owner_and_panel_boundaries():
    L = SU.make_layout(64, 96, 48, 8, b=16)          # 2 x 4 grid: k_c = 12, k_r = 24
    pcs = L.k_pieces()
    assert [p[0] for p in pcs] == [0, 12, 16, 24, 32, 36]
    assert sum(p[1] for p in pcs) == 48
    assert pcs[1] == (12, 4, 1, 0, 0, 12)            # A column 1 from 0, B row 0 from 12
    assert pcs[3] == (24, 8, 2, 0, 1, 0)
    for g, w, ac, ao, br, bo in pcs:
        assert ac * L.k_c + ao == g and br * L.k_r + bo == g
        assert ao + w <= L.k_c and bo + w <= L.k_r and g // L.b == (g + w - 1) // L.b
    assert SU.make_layout(32, 32, 32, 1, b=32).k_pieces() == [(0, 32, 0, 0, 0, 0)]


@pytest.mark.parametrize("P,b", [(1, 8), (2, 8), (4, 16), (8, 4), (8, 64)])
@pytest.mark.parametrize("direct", [True, False])
def test_p2p_schedule_matches_dense(P, b, direct):
    m, n, k = 48, 40, 64
    A, B, C = dense(m, n, k, 5)
    want = C - 0.25 * (A @ B)
    L = SU.make_layout(m, n, k, P, b=b)
    blocks = [SU.local_blocks(L, r, A, B, C) for r in range(P)]
    Ap, Bp = [a for a, _, _ in blocks], [bb for _, bb, _ in blocks]
    for r in range(P):
        c = blocks[r][2].clone()
        n_up = SU.summa_p2p(L, r, Ap, Bp, c, alpha=-0.25, local_gemm=matmul_update,
                            direct=direct)
        assert n_up == len(L.k_pieces())
        _, _, wc = SU.local_blocks(L, r, A, B, want)
        assert torch.allclose(c, wc, rtol=0, atol=1e-12)


def _colmajor_cuda(x):
    return x.t().contiguous().t().cuda()


@pytest.mark.gpu
@pytest.mark.parametrize("P,variant,level,b", [(2, "naive", 2, 2048), (4, "c", 2, 512),
                                               (8, "abc", 1, 256), (4, "ab", 2, 1024),
                                               (2, "dgemm", 0, 2048)])
def test_p2p_loopback_on_gpu_with_strassen_kernels(cuda, P, variant, level, b):
    """Peer-memory schedule with the real kernels reading strided views of the owners'
    blocks (direct for Naive/C, staged for the others)."""
    m, n, k = 1024, 2048, 2048
    A, B, C = (x.to(cuda) for x in dense(m, n, k, 9))
    L = SU.make_layout(m, n, k, P, b=b)
    blocks = [[_colmajor_cuda(x.cpu()) for x in SU.local_blocks(L, r, A, B, C)] for r in range(P)]
    Ap, Bp = [x[0] for x in blocks], [x[1] for x in blocks]
    want = C + A @ B
    an, bn = torch.linalg.norm(A).item(), torch.linalg.norm(B).item()
    for r in range(P):
        SU.summa_p2p(L, r, Ap, Bp, blocks[r][2], variant=variant, level=level)
        torch.cuda.synchronize()
        _, _, wc = SU.local_blocks(L, r, A, B, want)
        nw = (torch.linalg.norm(blocks[r][2] - wc) / (an * bn)).item()
        assert nw <= (1e-12 if level <= 1 else 5e-12), (r, nw)


def _ipc_worker(rank, world, port, variant, level, b, q):
    """One process of a world-2 job on ONE GPU: the peer block is a CUDA IPC mapping of
    the other process's memory, read by this process's kernels (no kernel waits on
    another process's kernel; the barriers order whole steps)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        m, n, k = 512, 1024, 1536
        A, B, C = dense(m, n, k, 21)
        L = SU.make_layout(m, n, k, world, b=b)
        a, bb, c = (_colmajor_cuda(x) for x in SU.local_blocks(L, rank, A, B, C))
        torch.cuda.synchronize()
        Ap, Bp = SU.open_peer_blocks(a, bb)
        dist.barrier()
        SU.summa_p2p(L, rank, Ap, Bp, c, variant=variant, level=level)
        torch.cuda.synchronize()
        dist.barrier()                      # peers are done reading this rank's blocks
        want = C + A @ B
        _, _, wc = SU.local_blocks(L, rank, A, B, want)
        nw = float(torch.linalg.norm(c.cpu() - wc) / (torch.linalg.norm(A) * torch.linalg.norm(B)))
        q.put((rank, nw, Ap[1 - rank].data_ptr() != a.data_ptr()))
        del Ap, Bp
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("variant,level,b", [("naive", 2, 1536), ("abc", 1, 512)])
def test_p2p_ipc_two_processes_one_gpu(cuda, variant, level, b):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, variant, level, b, q))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(2))
    for r, nw, mapped in res:
        assert mapped
        assert nw <= (1e-12 if level == 1 else 5e-12), (r, nw)
