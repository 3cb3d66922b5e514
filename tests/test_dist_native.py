"""The native distributed entry points (include/strassen_dist.h, csrc/dist.cpp): the
SUMMA schedule a C caller of the drop-in library reaches.  CPU: the schedule functions
against the Python layer's Layout, validation, and a C program compiled against the
header.  GPU: the 1 x 1 grid over NCCL, and whole grids through the loopback transport,
bitwise against the Python schedule and against the oracle."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest
import torch

import paper_1605_01078_b200 as S
from paper_1605_01078_b200 import summa as SU

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "dist_c_test")


def _build():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "capi")], check=True)


def test_every_symbol_of_the_dist_header_is_exported():
    src = open(os.path.join(ROOT, "include", "strassen_dist.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = sorted(set(re.findall(r"\b(strassen_dist_[a-z0-9_]+)\s*\(", src)))
    assert len(names) >= 15
    lib = C.CDLL(S.LIB_PATH)
    assert not [n for n in names if not hasattr(lib, n)]


def test_grid_and_default_panel_match_the_python_layer():
    for p in range(1, 33):
        assert SU.NativeGrid.grid(p) == SU.grid_for(p)
    for k in (1, 96, 8192, 16384, 65536, 46336, 92672, 3 * 8192):
        assert SU.NativeGrid.default_panel(k) == SU.make_layout(8, 8, k, 1).b


@pytest.mark.parametrize("P", [1, 2, 4, 6, 8, 16])
def test_panel_pieces_match_the_python_layer(P):
    pr, pc = SU.grid_for(P)
    k = 48 * pr * pc
    for b in [d for d in range(1, k + 1) if k % d == 0]:
        L = SU.make_layout(pr * 2, pc * 2, k, P, b=b)
        for p in range(L.panels):
            assert SU.NativeGrid.panel_pieces(k, pr, pc, b, p, "a") == L.a_pieces(p)
            assert SU.NativeGrid.panel_pieces(k, pr, pc, b, p, "b") == L.b_pieces(p)


def test_schedule_validation():
    with pytest.raises(S.StrassenError) as e:
        SU.NativeGrid.panel_pieces(48, 2, 4, 5, 0, "a")      # b does not divide k
    assert e.value.status == S.ERR_PARAM
    with pytest.raises(S.StrassenError):
        SU.NativeGrid.panel_pieces(50, 2, 4, 25, 0, "a")     # k does not divide the grid
    with pytest.raises(S.StrassenError):
        SU.NativeGrid.panel_pieces(48, 2, 4, 24, 2, "b")     # panel out of range
    with pytest.raises(S.StrassenError):
        SU.NativeGrid.grid(0)


def test_c_caller_of_the_dist_header_compiles_and_links():
    _build()
    r = subprocess.run([EXE, "--no-device"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout


# ------------------------------------------------------------------------- GPU
def _colmajor(x, dev, pad=0):
    """Column-major device copy with leading dimension rows + pad."""
    r, c = x.shape
    base = torch.zeros((c, r + pad), dtype=torch.float64, device=dev)
    v = base[:, :r].t()
    v.copy_(x)
    return v


def _dense(m, n, k, seed):
    g = torch.Generator().manual_seed(seed)
    return tuple(torch.rand(s, dtype=torch.float64, generator=g) * 2 - 1
                 for s in ((m, k), (k, n), (m, n)))


@pytest.mark.gpu
def test_c_caller_runs_nccl_and_loopback_grids_on_device(cuda):
    _build()
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
    assert r.stdout.count("nccl 1x1") == 2 and r.stdout.count("loopback") == 4


@pytest.mark.gpu
@pytest.mark.parametrize("variant,level,panel", [("abc", 2, 512), ("naive", 2, 0), ("dgemm", 0, 256)])
def test_nccl_single_rank_grid_bitwise_equals_the_rank_b_schedule(cuda, variant, level, panel):
    """1 x 1 grid over a real NCCL communicator (ncclCommInitRank + two ncclCommSplit):
    the result must be bitwise the reference bench's rank-b schedule
    (bench_lib.cpp:56-71) run through strassen_gemm_device on the same panels."""
    m, n, k = 1024, 768, 2048
    A, B, C0 = _dense(m, n, k, 31)
    a, b = _colmajor(A, cuda, pad=2), _colmajor(B, cuda)
    c1, c2 = _colmajor(C0, cuda), _colmajor(C0, cuda)
    ctx = S.Ctx()
    grid = SU.NativeGrid.nccl(ctx, SU.NativeGrid.unique_id(), 0, 1, 1, 1)
    assert grid.position() == (0, 1, 1, 0, 0)
    grid.gemm(variant, level, m, n, k, 0.5, a, b, c1, panel=panel)
    bw = panel or k
    assert grid.last_counts()[1] == k // bw
    for p0 in range(0, k, bw):
        ctx.gemm_device(variant, level, 0.5, a[:, p0:p0 + bw], b[p0:p0 + bw, :], c2)
    torch.cuda.synchronize()
    assert torch.equal(c1, c2)
    want = C0 + 0.5 * (A @ B)
    nw = (torch.linalg.norm(c1.cpu() - want) / (torch.linalg.norm(A) * torch.linalg.norm(B))).item()
    assert nw <= 5e-12
    grid.close()


@pytest.mark.gpu
@pytest.mark.parametrize("P,variant,level,b", [(2, "abc", 1, 256), (4, "abc", 2, 256),
                                               (8, "c", 2, 256), (8, "naive", 2, 2048),
                                               (4, "ab", 1, 1024)])
def test_native_loopback_bitwise_equals_the_python_schedule(cuda, P, variant, level, b):
    """Every rank of a grid through the native schedule on one GPU (record + replay
    passes of the loopback transport), against the Python summa_loopback with the same
    local kernels (bitwise) and against a dense product."""
    m, n, k = 1024, 2048, 2048
    A, B, C0 = (x.to(cuda) for x in _dense(m, n, k, 3))
    L = SU.make_layout(m, n, k, P, b=b)
    blocks = [SU.local_blocks(L, r, A, B, C0) for r in range(P)]
    Ab = [_colmajor(x[0], cuda) for x in blocks]
    Bb = [_colmajor(x[1], cuda, pad=4 * (r % 2)) for r, x in enumerate(blocks)]
    C_native = [_colmajor(x[2], cuda) for x in blocks]
    C_python = [_colmajor(x[2], cuda) for x in blocks]
    launches = SU.summa_native_loopback(L, Ab, Bb, C_native, alpha=-0.75, variant=variant,
                                        level=level)
    assert launches >= P * L.panels
    SU.summa_loopback(L, Ab, Bb, C_python, alpha=-0.75, variant=variant, level=level)
    torch.cuda.synchronize()
    want = C0 - 0.75 * (A @ B)
    an, bn = torch.linalg.norm(A).item(), torch.linalg.norm(B).item()
    for r in range(P):
        assert torch.equal(C_native[r], C_python[r]), r
        _, _, wc = SU.local_blocks(L, r, A, B, want)
        nw = (torch.linalg.norm(C_native[r] - wc) / (an * bn)).item()
        assert nw <= (1e-12 if level <= 1 else 5e-12), (r, nw)


@pytest.mark.gpu
def test_native_dist_gemm_is_stream_ordered_with_its_producers(cuda):
    """The blocks are produced on the caller's stream right before the call and changed
    right after it: the exchange steps must see the former and not the latter."""
    m, n, k = 512, 512, 1024
    A, B, C0 = _dense(m, n, k, 77)
    ctx = S.Ctx()
    grid = SU.NativeGrid.nccl(ctx, SU.NativeGrid.unique_id(), 0, 1, 1, 1)
    s = torch.cuda.Stream()
    a, b, c = _colmajor(A, cuda), _colmajor(B, cuda), _colmajor(C0, cuda)
    big = torch.empty(1 << 28, dtype=torch.float64, device=cuda)   # 2 GiB fill delays the stream
    a_late = torch.zeros_like(a)
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        big.fill_(1.0)
        a_late.copy_(a)                       # the real A arrives late on the stream
        grid.gemm("abc", 1, m, n, k, 1.0, a_late, b, c, panel=256, stream=s)
        a_late.zero_()                        # and is overwritten right after the call
    s.synchronize()
    want = C0 + A @ B
    nw = (torch.linalg.norm(c.cpu() - want) / (torch.linalg.norm(A) * torch.linalg.norm(B))).item()
    assert nw <= 1e-12
    grid.close()
