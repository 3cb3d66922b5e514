"""Narrow-tile launches (kernels.hpp kNarrowBN: 128 x 64 tiles, two CTAs per SM), which
the planner picks for small DGEMM / C / Naive problems (engine.cpp run_strassen): against
cuBLAS with the BASELINE normwise bounds, ragged and strided C, and -- forced on for every
variant through STRASSEN_B200_NARROW=1 in a child process (read once per process) -- the
fused-sum programs too, where sides longer than two terms are materialised."""
import os
import subprocess
import sys

import pytest

import paper_1605_01078_b200 as S

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _check(ctx, v, L, m, n, k, ld_pad, alpha, seed):
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    A = (torch.rand(k, m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    B = (torch.rand(n, k, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    big = torch.full((n, m + ld_pad), -5.5, dtype=torch.float64, device="cuda").t()
    C = big[:m, :]
    C.copy_((torch.rand(n, m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t())
    ref = C + alpha * (A @ B)
    ctx.gemm_device(v, L, alpha, A, B, C)
    torch.cuda.synchronize()
    nw = (torch.linalg.norm(C - ref) / (torch.linalg.norm(A) * torch.linalg.norm(B))).item()
    assert nw <= (5e-12 if L == 2 else 1e-12), (v, L, m, n, k, nw)
    if ld_pad:
        assert bool((big[m:, :] == -5.5).all())
    return C.clone()


@pytest.mark.parametrize("v,L,shape", [
    ("dgemm", 0, (1024, 1024, 1024)), ("dgemm", 0, (1000, 777, 1030)), ("dgemm", 0, (64, 8000, 300)),
    ("c", 1, (1024, 1024, 1024)), ("c", 2, (2048, 2048, 2048)), ("c", 2, (1281, 1999, 1100)),
    ("naive", 1, (1000, 1000, 1000)), ("naive", 2, (1024, 1536, 700)),
])
@pytest.mark.parametrize("ld_pad", [0, 3])
def test_narrow_planned_sizes(cuda, v, L, shape, ld_pad):
    """Sizes the planner runs with narrow tiles: BASELINE bounds, ld padding untouched
    (odd ldc: the scalar epilogue), and a repeated call is bitwise repeatable."""
    import torch
    m, n, k = shape
    ctx = S.Ctx()
    first = _check(ctx, v, L, m, n, k, ld_pad, 1.0 if ld_pad else -0.5, seed=m + n + k)
    second = _check(ctx, v, L, m, n, k, ld_pad, 1.0 if ld_pad else -0.5, seed=m + n + k)
    assert torch.equal(first, second)
    ctx.close()


_CHILD = r"""
import sys, torch
sys.path.insert(0, {root!r})
import paper_1605_01078_b200 as S
ctx = S.Ctx()
worst = 0.0
for v, L, m, n, k in [("abc", 1, 1024, 1024, 1024), ("abc", 2, 2048, 2048, 2048), ("ab", 1, 1000, 1100, 900),
                      ("ab", 2, 1536, 1024, 1280), ("abc", 2, 777, 1030, 513), ("naive", 2, 2048, 2048, 1024),
                      ("dgemm", 0, 3000, 2000, 1500), ("c", 1, 4096, 4096, 256)]:
    for f in (4, 2):
        ctx.set_fused_terms(f)
        g = torch.Generator(device="cuda").manual_seed(m * n + k)
        A = (torch.rand(k, m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
        B = (torch.rand(n, k, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
        C = (torch.rand(n, m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
        ref = C + A @ B
        ctx.gemm_device(v, L, 1.0, A, B, C)
        torch.cuda.synchronize()
        nw = (torch.linalg.norm(C - ref) / (torch.linalg.norm(A) * torch.linalg.norm(B))).item()
        assert nw <= (5e-12 if L == 2 else 1e-12), (v, L, m, n, k, f, nw)
        if f == 4:
            keep = C.clone()
        else:
            assert torch.equal(C, keep), (v, L, m, n, k)
        worst = max(worst, nw)
print("narrow forced ok", worst)
"""


def test_narrow_forced_on_every_variant(cuda):
    """STRASSEN_B200_NARROW=1: every variant (fused-sum ones included, their 4-term sides
    materialised) within the bounds, and the fused-term setting still bitwise neutral."""
    env = dict(os.environ, STRASSEN_B200_NARROW="1")
    out = subprocess.run([sys.executable, "-c", _CHILD.format(root=ROOT)], env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    assert "narrow forced ok" in out.stdout


_COOP_CHILD = r"""
import hashlib, sys, torch
sys.path.insert(0, {root!r})
import paper_1605_01078_b200 as S
ctx = S.Ctx()
for v, L, m, n, k, row_major in [("dgemm", 0, 768, 768, 768, 0), ("dgemm", 0, 896, 896, 896, 0),
                                 ("dgemm", 0, 768, 640, 2048, 1), ("dgemm", 0, 777, 1031, 515, 0),
                                 ("dgemm", 0, 777, 1031, 515, 1), ("dgemm", 0, 1024, 1024, 1024, 0),
                                 ("abc", 1, 1024, 1024, 1024, 0), ("c", 1, 1000, 1000, 1000, 0),
                                 ("naive", 1, 1280, 1280, 1280, 1), ("dgemm", 0, 2048, 2048, 2048, 0)]:
    g = torch.Generator(device="cuda").manual_seed(m + 3 * n + 7 * k)
    A = (torch.rand(k, m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    B = (torch.rand(n, k, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    C0 = (torch.rand(n, m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    ref = C0 + A @ B
    out = []
    for rep in range(2):
        C = C0.contiguous().clone() if row_major else C0.t().clone().t()
        ctx.gemm_device(v, L, 1.0, A, B, C)
        torch.cuda.synchronize()
        nw = (torch.linalg.norm(C - ref) / (torch.linalg.norm(A) * torch.linalg.norm(B))).item()
        assert nw <= 1e-12, (v, L, m, n, k, nw)
        out.append(hashlib.sha1(C.contiguous().cpu().numpy().tobytes()).hexdigest())
    assert out[0] == out[1], "not repeatable"
    print("sum", v, L, m, n, k, row_major, out[0])
print("coop child ok")
"""


def test_cooperative_fixup_bitwise_equal_to_single_owner(cuda):
    """The cooperative k-split fixup (kernels.hpp MMParams::coop_fixup: the pieces of a
    tile share the sum of the partials and the C update) gives bit for bit the
    single-owner fixup's result -- same piece order per element -- on k-chunk grids
    (default) and on stream-K launches (STRASSEN_B200_COOP_SK=1), within the BASELINE
    bound of cuBLAS and repeatably; column- and row-major C (vector / scalar updates)."""
    sums = {}
    for name, extra in [("off", {"STRASSEN_B200_COOP": "0"}), ("on", {"STRASSEN_B200_COOP": "1"}),
                        ("on+sk", {"STRASSEN_B200_COOP": "1", "STRASSEN_B200_COOP_SK": "1"})]:
        out = subprocess.run([sys.executable, "-c", _COOP_CHILD.format(root=ROOT)],
                             env=dict(os.environ, **extra), capture_output=True, text=True,
                             timeout=600)
        assert out.returncode == 0, (name, out.stderr[-3000:])
        assert "coop child ok" in out.stdout
        sums[name] = [ln for ln in out.stdout.splitlines() if ln.startswith("sum ")]
        assert len(sums[name]) == 10
    assert sums["off"] == sums["on"] == sums["on+sk"]


@pytest.mark.parametrize("shape", [(2304, 2304, 2304), (2816, 2432, 700), (2301, 2417, 777),
                                   (3000, 3000, 520)])
def test_classical_stream_k_between_two_and_four_waves(cuda, shape):
    """Classical launches of two to four waves of 128 x 128 tiles run stream-K over all
    the tiles instead of whole waves of tile owners (engine.cpp plan_fused): within the
    BASELINE bound of cuBLAS, repeatable, and the host-pointer call (never windowed under
    four waves) bitwise equal to the device call."""
    import numpy as np
    import torch
    m, n, k = shape
    ctx = S.Ctx()
    first = _check(ctx, "dgemm", 0, m, n, k, 0, -0.5, seed=m + n + k)
    second = _check(ctx, "dgemm", 0, m, n, k, 0, -0.5, seed=m + n + k)
    assert torch.equal(first, second)
    g = torch.Generator(device="cuda").manual_seed(m + n + k)
    A = (torch.rand(k, m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    B = (torch.rand(n, k, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    C0 = (torch.rand(n, m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    a, b = np.asfortranarray(A.cpu().numpy()), np.asfortranarray(B.cpu().numpy())
    c = np.asfortranarray(C0.cpu().numpy())
    ctx.gemm("dgemm", 0, -0.5, a, b, c)              # host pointers through strassen_gemm
    assert np.array_equal(c, first.cpu().numpy())
    ctx.close()


@pytest.mark.parametrize("shape", [(3328, 3328, 2048), (3840, 3840, 1030), (3333, 3841, 1100),
                                   (5632, 5632, 1024)])
def test_classical_tile_owner_waves_plus_stream_k_tail(cuda, shape):
    """Classical launches from four waves of tiles up: whole waves of tile owners on the
    first tile columns, stream-K pieces on the last ones (plan.hpp choose_tail) -- two
    launches; within the BASELINE bound of cuBLAS, repeatable, and the unpipelined
    host-pointer call bitwise equal to the device call."""
    import numpy as np
    import torch
    m, n, k = shape
    ctx = S.Ctx()
    first = _check(ctx, "dgemm", 0, m, n, k, 0, -0.5, seed=m + n + k)
    assert ctx.last_launches() >= 2
    second = _check(ctx, "dgemm", 0, m, n, k, 0, -0.5, seed=m + n + k)
    assert torch.equal(first, second)
    g = torch.Generator(device="cuda").manual_seed(m + n + k)
    A = (torch.rand(k, m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    B = (torch.rand(n, k, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    C0 = (torch.rand(n, m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    a, b = np.asfortranarray(A.cpu().numpy()), np.asfortranarray(B.cpu().numpy())
    c = np.asfortranarray(C0.cpu().numpy())
    ctx.set_pipelining(False)
    ctx.gemm("dgemm", 0, -0.5, a, b, c)              # host pointers, one window
    assert np.array_equal(c, first.cpu().numpy())
    # the pipelined host call keeps the plain tile-owner grid (its windows cannot run a
    # whole call's pieces): same bound
    ctx.set_pipelining(True)
    c2 = np.asfortranarray(C0.cpu().numpy())
    ctx.gemm("dgemm", 0, -0.5, a, b, c2)
    ref = (C0 - 0.5 * (A @ B)).cpu().numpy()
    nw = np.linalg.norm(c2 - ref) / (np.linalg.norm(a) * np.linalg.norm(b))
    assert nw <= 1e-12
    ctx.close()
