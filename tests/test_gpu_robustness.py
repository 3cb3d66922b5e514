"""Robustness of the B200 path (through the C ABI): fused-term settings, the dynamic
unit hand-out of persistent launches under SM contention, ctx workspace ordering
across streams, operand events on the windowed host path and the device entry's
host-pointer rejection.  Checked against cuBLAS (fp64 torch matmul) with the
BASELINE normwise bounds, and bitwise where the arithmetic is the same."""
import numpy as np
import pytest

import paper_1605_01078_b200 as S
from gpu_util import inputs

pytestmark = pytest.mark.gpu


def _dev(m, n, k, seed):
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    A = (torch.rand(k, m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    B = (torch.rand(n, k, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    C0 = (torch.rand(n, m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    return A, B, C0


def _clone(X):
    return X.clone().t().contiguous().t()


def _normwise(C, ref, A, B):
    import torch
    return (torch.linalg.norm(C - ref) / (torch.linalg.norm(A) * torch.linalg.norm(B))).item()


@pytest.mark.parametrize("variant,level", [("abc", 1), ("abc", 2), ("ab", 1), ("ab", 2)])
@pytest.mark.parametrize("shape", [(1000, 1000, 1000), (2048, 2048, 2048), (4100, 3000, 2050),
                                   (8192, 8192, 1024)])
def test_fused_terms_bitwise_identical(cuda, variant, level, shape):
    """strassen_ctx_set_fused_terms: sides summed in registers or materialised by the
    sum pass add the same terms in the same order -- every setting gives the same
    bits (and the BASELINE bound against cuBLAS)."""
    import torch
    m, n, k = shape
    A, B, C0 = _dev(m, n, k, seed=m + 7 * n + 13 * k)
    ref = C0 + A @ B
    first = None
    for f in (4, 3, 2, 1):
        ctx = S.Ctx()
        ctx.set_fused_terms(f)
        C = _clone(C0)
        ctx.gemm_device(variant, level, 1.0, A, B, C)
        torch.cuda.synchronize()
        ctx.close()
        if first is None:
            first = C
            assert _normwise(C, ref, A, B) <= (5e-12 if level == 2 else 1e-12)
        else:
            assert torch.equal(C, first), (variant, level, shape, f)


def test_fused_terms_host_windows(cuda):
    """The host-call window pipeline with materialised 4-term sides (ABC L2, default
    setting) equals the device entry bitwise."""
    import torch
    d = 6144
    a, b, c0 = inputs(d, d, d, (41, 42, 43))
    ctx = S.Ctx()
    host = np.array(c0, order="F")
    ctx.gemm("abc", 2, 1.0, a, b, host)
    ta, tb = (torch.from_numpy(np.ascontiguousarray(x.T)).cuda().t() for x in (a, b))
    tc = torch.from_numpy(np.ascontiguousarray(c0.T)).cuda().t()
    ctx.set_fused_terms(4)
    ctx.gemm_device("abc", 2, 1.0, ta, tb, tc)
    torch.cuda.synchronize()
    assert np.array_equal(tc.cpu().numpy(), host)
    ctx.close()


def test_fused_terms_rejects_out_of_range():
    ctx = S.Ctx()
    for bad in (0, 5, -1):
        with pytest.raises(S.StrassenError):
            ctx.set_fused_terms(bad)
    assert S.lib().strassen_ctx_set_fused_terms(None, 2) == S.ERR_NULL
    ctx.close()


@pytest.mark.parametrize("variant,level", [("naive", 2), ("c", 2), ("c", 1), ("dgemm", 0)])
def test_persistent_launch_with_sms_held_by_another_kernel(cuda, variant, level):
    """A persistent mm launch (one CTA per SM) whose SMs are partly held by kernels
    launched just before it on other streams (as a co-scheduled NCCL broadcast would):
    the late CTAs take fewer units from the dynamic counter; the result is bitwise
    that of an undisturbed call, and the call is not delayed by the whole sleep."""
    import torch
    d = 8192
    A, B, C0 = _dev(d, d, d, seed=81)
    ctx = S.Ctx()
    solo = _clone(C0)
    ctx.gemm_device(variant, level, 1.0, A, B, solo)
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(40)]
    C = _clone(C0)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    for st in streams:
        with torch.cuda.stream(st):
            torch.cuda._sleep(50_000_000)  # ~25 ms on one SM each
    t0.record()
    ctx.gemm_device(variant, level, 1.0, A, B, C)
    t1.record()
    torch.cuda.synchronize()
    assert torch.equal(C, solo), (variant, level)
    print(f"{variant}{level} 8192^3 with 40 SMs held ~25 ms: {t0.elapsed_time(t1):.1f} ms")
    ctx.close()


def test_ctx_calls_on_two_streams_are_ordered(cuda):
    """Two back-to-back calls on one ctx, each on its own stream: the second must not
    overwrite the shared workspace (operand sums, product temporaries, tickets) while
    the first call's kernels still read it (gemm_impl orders a call after the last)."""
    import torch
    d = 4096
    A1, B1, C1 = _dev(d, d, d, seed=1)
    A2, B2, C2 = _dev(d, d, d, seed=2)
    ref1, ref2 = C1 + A1 @ B1, C2 + A2 @ B2
    ctx = S.Ctx()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for v, L in [("naive", 2), ("c", 2), ("abc", 2), ("ab", 1)]:
        X1, X2 = _clone(C1), _clone(C2)
        torch.cuda.synchronize()
        ctx.gemm_device(v, L, 1.0, A1, B1, X1, stream=s1)
        ctx.gemm_device(v, L, 1.0, A2, B2, X2, stream=s2)
        torch.cuda.synchronize()
        assert _normwise(X1, ref1, A1, B1) <= 5e-12, (v, L, 1)
        assert _normwise(X2, ref2, A2, B2) <= 5e-12, (v, L, 2)
    ctx.close()


def test_windowed_host_call_waits_for_late_device_a(cuda):
    """Host B and C (window pipeline) with a device A still being produced on another
    stream (strassen_ctx_set_operand_events): the windows must wait for A."""
    import torch
    d = 6144
    _, b, c0 = inputs(d, d, d, (51, 52, 53))
    A0 = (torch.rand(d, d, dtype=torch.float64, device="cuda") * 2 - 1).t()
    ref = torch.from_numpy(np.ascontiguousarray(c0.T)).cuda().t() + \
        A0 @ torch.from_numpy(np.ascontiguousarray(b.T)).cuda().t()
    A = torch.zeros((d, d), dtype=torch.float64, device="cuda").t()  # stale
    side = torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(side):
        torch.cuda._sleep(60_000_000)
        A.copy_(A0)
        ev = torch.cuda.Event()
        ev.record(side)
    ctx = S.Ctx()
    ctx.set_operand_events(a=ev)
    c = np.array(c0, order="F")
    ctx.gemm("naive", 2, 1.0, A, b, c)
    got = torch.from_numpy(np.ascontiguousarray(c.T)).cuda().t()
    assert _normwise(got, ref, A0, torch.from_numpy(b).cuda()) <= 5e-12
    ctx.close()


def test_device_entry_rejects_host_operands_before_staging(cuda):
    """strassen_gemm_device with a host pointer: STRASSEN_ERR_PARAM, and no staging
    buffer was grown on the way."""
    import torch
    d = 2048
    A, B, _ = _dev(d, d, d, seed=3)
    c = np.zeros((d, d), order="F")
    ctx = S.Ctx()
    with pytest.raises(S.StrassenError) as ei:
        ctx.gemm_device("naive", 2, 1.0, A, B, c)
    assert ei.value.status == S.ERR_PARAM
    assert ctx.workspace_bytes() == 0
    ctx.close()


@pytest.mark.parametrize("variant,level", [("abc", 1), ("abc", 2), ("c", 1), ("c", 2)])
@pytest.mark.parametrize("shape", [(6144, 6144, 512), (4117, 4100, 1030), (3000, 5000, 256)])
def test_product_groups_in_tensor_memory(cuda, variant, level, shape):
    """Short products of ABC / C run in groups of up to three per unit (the first ones
    parked in TMEM) with one combined update per destination: against cuBLAS, bitwise
    repeatable, and bitwise the same whether C takes the TMA reduce-add epilogue (even
    ldc) or the register path (odd ldc) -- alpha = 1, where both round once."""
    import torch
    m, n, k = shape
    A, B, C0 = _dev(m, n, k, seed=m + n + k + level)
    ref = C0 + A @ B
    ctx = S.Ctx()
    outs = []
    for ld in (m + (m & 1), m + (m & 1), m | 1):  # even ldc twice, then odd ldc
        big = torch.zeros((n, ld), dtype=torch.float64, device="cuda").t()
        C = big[:m, :]
        C.copy_(C0)
        ctx.gemm_device(variant, level, 1.0, A, B, C)
        torch.cuda.synchronize()
        outs.append(C.clone())
    ctx.close()
    assert _normwise(outs[0], ref, A, B) <= (5e-12 if level == 2 else 1e-12)
    assert torch.equal(outs[0], outs[1])
    assert torch.equal(outs[0], outs[2]), (variant, level, shape)


@pytest.mark.parametrize("variant,level,shape", [
    ("dgemm", 0, (512, 512, 512)), ("dgemm", 0, (1024, 1024, 1024)), ("abc", 1, (1024, 1024, 1024)),
    ("c", 1, (1000, 900, 1100)), ("abc", 2, (2048, 2048, 2048)), ("naive", 2, (2048, 1536, 1024)),
    ("ab", 2, (1536, 1536, 1536)), ("c", 2, (4096, 4096, 512)),
    ("dgemm", 0, (3840, 3840, 1030)),   # tile-owner waves + stream-K tail (two launches)
    ("c", 2, (4100, 4100, 520)),        # peeled to whole tiles: fringe kernels
    ("dgemm", 0, (768, 768, 768)),      # k-chunk grid, cooperative fixup
])
def test_device_entry_under_cuda_graph_capture(cuda, variant, level, shape):
    """strassen_gemm_device issued on a capturing stream (include/strassen.h): the call's
    launches and counter resets become graph nodes; replays are bitwise equal to the eager
    call, repeatably, and within the BASELINE bound of cuBLAS."""
    import torch
    m, n, k = shape
    A, B, C0 = _dev(m, n, k, seed=m + n + k)
    ctx = S.Ctx()
    Ce = _clone(C0)
    ctx.gemm_device(variant, level, 1.0, A, B, Ce)   # eager; also sizes the workspace
    torch.cuda.synchronize()
    ref = C0 + A @ B
    assert _normwise(Ce, ref, A, B) <= (5e-12 if level == 2 else 1e-12)
    Cg = _clone(C0)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        ctx.gemm_device(variant, level, 1.0, A, B, Cg, torch.cuda.current_stream())
    for _ in range(3):
        Cg.copy_(C0)
        graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(Cg, Ce)
    # eager calls on the same ctx still work after the capture
    Ce2 = _clone(C0)
    ctx.gemm_device(variant, level, 1.0, A, B, Ce2)
    torch.cuda.synchronize()
    assert torch.equal(Ce2, Ce)
    ctx.close()


def test_capture_that_would_grow_the_workspace_is_refused(cuda):
    """A captured call may not grow the ctx's workspace (growing synchronises the
    device): STRASSEN_ERR_ALLOC before any CUDA call that would invalidate the capture,
    and the ctx works again afterwards."""
    import torch
    A, B, C0 = _dev(512, 512, 512, seed=5)
    A2, B2, C2 = _dev(2048, 2048, 2048, seed=6)
    ctx = S.Ctx()
    C = _clone(C0)
    ctx.gemm_device("naive", 1, 1.0, A, B, C)        # initialises the ctx, small workspace
    torch.cuda.synchronize()
    Cg = _clone(C2)
    graph = torch.cuda.CUDAGraph()
    with pytest.raises(S.StrassenError) as ei:
        with torch.cuda.graph(graph):
            ctx.gemm_device("naive", 2, 1.0, A2, B2, Cg, torch.cuda.current_stream())
    assert ei.value.status == S.ERR_ALLOC and "capture" in str(ei.value)
    torch.cuda.synchronize()
    Ce = _clone(C2)
    ctx.gemm_device("naive", 2, 1.0, A2, B2, Ce)     # eager: grows the workspace, runs
    torch.cuda.synchronize()
    assert _normwise(Ce, C2 + A2 @ B2, A2, B2) <= 5e-12
    ctx.close()
