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
