"""BASELINE config 5 at full size on ONE GPU: SUMMA m = n = k = 65536 over a 2 x 4 grid
of virtual ranks (summa_loopback: each "broadcast" is a device copy, ranks run one after
another), local two-level ABC Strassen updates, checked against the oracle on sampled
256 x 256 output tiles regenerated from the counter-based RNG (SURVEY.md §8c protocol 3),
plus an fp64 Freivalds check of the whole product.

usage: python tools/cfg5_loopback.py [N=65536] [P=8] [variant=abc] [level=2]
Prints one JSON line.  Needs ~110 GB of device memory at N = 65536.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch

import oracle_lib as O  # checker only
from gpu_util import counter_uniform_np, counter_uniform_torch
from paper_1605_01078_b200 import summa as SU


def run(N=65536, P=8, variant="abc", level=2, tiles=None, seed=5):
    torch.cuda.set_device(0)
    dev = "cuda"
    A = counter_uniform_torch(1, 0, N, 0, N, seed, dev)
    B = counter_uniform_torch(2, 0, N, 0, N, seed, dev)
    C = counter_uniform_torch(3, 0, N, 0, N, seed, dev)
    # the GPU generator agrees with the oracle-side one
    probe = counter_uniform_np(1, N - 37, 37, N - 41, 41, seed)
    assert np.array_equal(A[N - 37:, N - 41:].cpu().numpy(), probe)
    L = SU.make_layout(N, N, N, P)
    blocks = [SU.local_blocks(L, r, A, B, C) for r in range(P)]  # views: C updated in place
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    launches = SU.summa_loopback(L, [a for a, _, _ in blocks], [b for _, b, _ in blocks],
                                 [c for _, _, c in blocks], 1.0, variant, level)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    # fp64 Freivalds on the device: C x - C0 x - A (B x), C0 regenerated in column chunks
    g = torch.Generator(device=dev).manual_seed(seed)
    x = torch.rand((N, 1), dtype=torch.float64, device=dev, generator=g) * 2 - 1
    c0x = torch.zeros((N, 1), dtype=torch.float64, device=dev)
    for cs in range(0, N, 4096):
        ch = counter_uniform_torch(3, 0, N, cs, min(4096, N - cs), seed, dev)
        c0x += ch @ x[cs:cs + ch.shape[1]]
    r = C @ x - c0x - A @ (B @ x)
    frei = (torch.linalg.norm(r) / (torch.linalg.norm(A) * torch.linalg.norm(B) *
                                    torch.linalg.norm(x))).item()
    # sampled tiles against the oracle (block and panel boundaries included)
    tol = 1e-12 if level <= 1 else 5e-12
    tiles = tiles or [(0, 0), (L.m_l - 128, L.n_l - 128), (N - 256, N // 2 + 77)]
    errs = []
    for r0, c0 in tiles:
        a = counter_uniform_np(1, r0, 256, 0, N, seed)
        b = counter_uniform_np(2, 0, N, c0, 256, seed)
        c0h = counter_uniform_np(3, r0, 256, c0, 256, seed)
        ref = np.array(c0h, order="F")
        O.strassen_gemm("dgemm", 0, 1.0, a, b, ref)
        got = C[r0:r0 + 256, c0:c0 + 256].cpu().numpy()
        errs.append(O.normwise_error(got, ref, a, b))
    out = {"config": f"SUMMA m=n=k={N} on {L.pr}x{L.pc} virtual ranks (one GPU, loopback)",
           "variant": variant, "level": level, "panel_b": L.b,
           "local_update": [L.m_l, L.n_l, L.b], "local_calls": P * L.panels,
           "ms": ms, "effective_tflops_one_gpu": 2.0 * N ** 3 / (ms * 1e-3) / 1e12,
           "gpu_launches": launches, "freivalds_fp64": frei,
           "sampled_tile_normwise": errs, "tolerance": tol,
           "pass": bool(max(errs) <= tol and frei < 1e-13)}
    return out


if __name__ == "__main__":
    a = sys.argv[1:]
    res = run(int(a[0]) if a else 65536, int(a[1]) if len(a) > 1 else 8,
              a[2] if len(a) > 2 else "abc", int(a[3]) if len(a) > 3 else 2)
    print(json.dumps(res), flush=True)
    sys.exit(0 if res["pass"] else 1)
