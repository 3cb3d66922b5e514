"""SUMMA distributed layer: Strassen DGEMM sharded over the GPUs of one node.

The paper's distributed experiment runs SUMMA on a 2-D process grid,
with local one/two-level ABC Strassen as the rank-b update. The reference stops at an
in-process rank-b schedule (tools/bench_lib.cpp:56-71). SURVEY.md §8(e) is the
design followed here.

* Process grid pr x pc, chosen by :func:`grid_for` (P=2 -> 1x2, 4 -> 2x2, 8 -> 2x4).
  Rank r sits at (r // pc, r % pc).
* 2-D block distribution. Rank (i, j) owns
  A_ij = A[i*m_l:(i+1)*m_l, j*k_c:(j+1)*k_c]   (m_l = m/pr, k_c = k/pc)
  B_ij = B[i*k_r:(i+1)*k_r, j*n_l:(j+1)*n_l]   (k_r = k/pr, n_l = n/pc)
  C_ij = C[i*m_l:(i+1)*m_l, j*n_l:(j+1)*n_l]
* One exchange step per k-panel p of width b:
  * the rank(s) in process row i owning A columns [p*b, (p+1)*b) broadcast their
    m_l x w pieces along row i (one broadcast per owner when the panel straddles
    the k_c = k/pc columns a rank owns);
  * the rank(s) in process column j owning B rows [p*b, (p+1)*b) broadcast their
    w x n_l pieces along column j.
  Then every rank runs C_ij += alpha * A_panel @ B_panel locally, with the chosen variant
  and level (strassen_gemm_device on the current CUDA stream).
* Broadcasts for panel p+1 are issued asynchronously before the local update of panel p,
  into the other of two panel buffers, so communication overlaps compute.

Communicators:

* :class:`TorchComm` uses torch.distributed with one process per GPU. Row and column
  groups come from ``new_group``. NCCL runs over NVLink/NVSwitch; gloo runs on CPU for the
  tests.
* :func:`summa_p2p` is the same product with no broadcasts: every rank maps the other
  ranks' A and B blocks (:func:`open_peer_blocks`, CUDA IPC) and its local Strassen call
  reads the owners' memory directly.  For Naive and C the operand-sum pass is the only
  reader of A and B, so the gather over NVLink is fused into that pass; ABC, AB and the
  classical kernel re-read operand tiles, so their pieces are pulled by a side stream
  into a local double buffer first.
* :func:`summa_loopback` runs P virtual ranks in ONE process. Each "broadcast" is a device
  copy and the ranks execute one after another. It exercises the full data path and the
  real kernels on a single GPU; nothing waits on another launch.

The local update is pluggable (``local_gemm``), so the host-side distribution logic can be
checked on CPU against a dense product.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, List, Optional

import torch


def grid_for(p: int):
    """Most-square pr x pc grid with pr <= pc (1x2, 2x2, 2x4)."""
    pr = int(math.isqrt(p))
    while p % pr:
        pr -= 1
    return pr, p // pr


@dataclass
class Layout:
    m: int
    n: int
    k: int
    pr: int
    pc: int
    b: int  # panel width

    @property
    def m_l(self):
        return self.m // self.pr

    @property
    def n_l(self):
        return self.n // self.pc

    @property
    def k_c(self):  # A columns per rank
        return self.k // self.pc

    @property
    def k_r(self):  # B rows per rank
        return self.k // self.pr

    @property
    def panels(self):
        return self.k // self.b

    def a_owner_col(self, p):
        """Process column owning the first column of A panel p, and its local offset."""
        g = p * self.b
        return g // self.k_c, g % self.k_c

    def b_owner_row(self, p):
        g = p * self.b
        return g // self.k_r, g % self.k_r

    @staticmethod
    def _pieces(g0, width, per_owner):
        """Split global k range [g0, g0+width) at owner boundaries (multiples of per_owner):
        a list of (owner, local offset, piece width, offset inside the panel)."""
        out, g = [], g0
        while g < g0 + width:
            owner, off = divmod(g, per_owner)
            w = min(per_owner - off, g0 + width - g)
            out.append((owner, off, w, g - g0))
            g += w
        return out

    def a_pieces(self, p):
        """A panel p by owning process column: (col, local col offset, width, panel offset)."""
        return self._pieces(p * self.b, self.b, self.k_c)

    def b_pieces(self, p):
        """B panel p by owning process row: (row, local row offset, width, panel offset)."""
        return self._pieces(p * self.b, self.b, self.k_r)

    def k_pieces(self):
        """The k range cut at A-owner (k_c), B-owner (k_r) and panel (b) boundaries, for the
        peer-memory schedule: (g0, w, a_col, a_off, b_row, b_off) means A columns
        [a_off, a_off + w) of process column a_col times B rows [b_off, b_off + w) of
        process row b_row."""
        out, g = [], 0
        while g < self.k:
            ac, ao = divmod(g, self.k_c)
            br, bo = divmod(g, self.k_r)
            end = min((ac + 1) * self.k_c, (br + 1) * self.k_r, (g // self.b + 1) * self.b)
            out.append((g, end - g, ac, ao, br, bo))
            g = end
        return out


def make_layout(m, n, k, p, b=None):
    """Panels may straddle owner boundaries: a panel is then assembled from one broadcast
    per owning piece, so the panel width (the local update's k) is not capped by the
    k / pc columns of A a rank owns.  Default b: k halved while above 8192 (16384^2 local
    updates: naive L2 45.0 TF/s at k = 8192 against 43.5 at 4096, profiles/r01_sweep_rankk.csv,
    with one 1 GB panel broadcast exposed)."""
    pr, pc = grid_for(p)
    if m % pr or n % pc or k % pr or k % pc:
        raise ValueError(f"m={m}, n={n}, k={k} must divide the {pr}x{pc} grid")
    if b is None:
        b = k
        while b > 8192 and b % 2 == 0:  # bound the panel buffers
            b //= 2
    if b < 1 or k % b:
        raise ValueError(f"panel width {b} must divide k = {k}")
    return Layout(m, n, k, pr, pc, b)


def local_blocks(layout: Layout, rank: int, A: torch.Tensor, B: torch.Tensor, C: torch.Tensor):
    """Slices of global A, B, C owned by `rank` (for tests and data set-up)."""
    i, j = divmod(rank, layout.pc)
    a = A[i * layout.m_l:(i + 1) * layout.m_l, j * layout.k_c:(j + 1) * layout.k_c]
    b = B[i * layout.k_r:(i + 1) * layout.k_r, j * layout.n_l:(j + 1) * layout.n_l]
    c = C[i * layout.m_l:(i + 1) * layout.m_l, j * layout.n_l:(j + 1) * layout.n_l]
    return a, b, c


# ------------------------------------------------------------- communicators
class TorchComm:
    """torch.distributed (NCCL on GPUs, gloo on CPU) with row/column groups."""

    def __init__(self, layout: Layout):
        import torch.distributed as dist
        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        if self.world != layout.pr * layout.pc:
            raise ValueError("world size does not match the process grid")
        self.layout = layout
        self.i, self.j = divmod(self.rank, layout.pc)
        # every rank must create every group, in the same order
        self.row_groups = [dist.new_group([r * layout.pc + c for c in range(layout.pc)])
                           for r in range(layout.pr)]
        self.col_groups = [dist.new_group([r * layout.pc + c for r in range(layout.pr)])
                           for c in range(layout.pc)]

    def bcast_row(self, t: torch.Tensor, src_col: int):
        """Broadcast along this rank's process row from column src_col (async)."""
        if self.layout.pc == 1:
            return None
        return self.dist.broadcast(t, src=self.i * self.layout.pc + src_col,
                                   group=self.row_groups[self.i], async_op=True)

    def bcast_col(self, t: torch.Tensor, src_row: int):
        if self.layout.pr == 1:
            return None
        return self.dist.broadcast(t, src=src_row * self.layout.pc + self.j,
                                   group=self.col_groups[self.j], async_op=True)


def _default_local_gemm(variant, level):
    import paper_1605_01078_b200 as S
    ctx = S.Ctx()
    if level == 3:
        ctx.set_max_level(3)

    def run(alpha, a, b, c):
        if run.c_ready is not None:  # C still arriving: kernels wait right before reading it
            ctx.set_operand_events(c=run.c_ready)
            run.c_ready = None
        if c.is_cuda:
            ctx.gemm_device(variant, level, alpha, a, b, c)
        else:
            ctx.gemm(variant, level, alpha, a, b, c)
        return ctx.last_launches()
    run.ctx = ctx  # for profiling one local update (bench.py roofline at N > 1)
    run.c_ready = None  # torch.cuda.Event the next local update's C reads wait on
    return run


def summa(layout: Layout, comm: TorchComm, A_l: torch.Tensor, B_l: torch.Tensor,
          C_l: torch.Tensor, alpha: float = 1.0, variant="abc", level=1,
          local_gemm: Optional[Callable] = None) -> int:
    """C_l += alpha * (A @ B)_ij on rank (i, j) of a torch.distributed job.

    A_l (m_l x k_c), B_l (k_r x n_l), C_l (m_l x n_l) are the rank's blocks. The panel
    buffers are column-major, so the local Strassen call reads them through TMA without a
    repack. Returns the GPU kernel launches of the local updates (one per update when
    `local_gemm` reports no count).
    """
    L = layout
    gemm = local_gemm or _default_local_gemm(variant, level)
    dev = C_l.device

    # contiguous storage for the collectives, column-major views for the kernels
    abase = [torch.empty((L.b, L.m_l), dtype=torch.float64, device=dev) for _ in range(2)]
    bbase = [torch.empty((L.n_l, L.b), dtype=torch.float64, device=dev) for _ in range(2)]
    abuf = [t.t() for t in abase]
    bbuf = [t.t() for t in bbase]

    def post(p):
        """Issue panel p's broadcasts into buffer p % 2.  Returns the pending works and the
        B pieces that arrive in contiguous staging (a B panel straddling process rows:
        its row pieces are strided in the column-major panel) to be placed after the wait."""
        s = p % 2
        works, fixups = [], []
        for oc, lo, w, po in L.a_pieces(p):   # column pieces: contiguous in abase
            if comm.j == oc:
                abuf[s][:, po:po + w].copy_(A_l[:, lo:lo + w])
            works.append(comm.bcast_row(abase[s][po:po + w], oc))
        pieces = L.b_pieces(p)
        for idx, (orow, lo, w, po) in enumerate(pieces):
            if len(pieces) == 1:
                dst = bbase[s]
                if comm.i == orow:
                    bbuf[s].copy_(B_l[lo:lo + w, :])
            else:
                key = (s, idx, w)
                if key not in bstage:
                    bstage[key] = torch.empty((L.n_l, w), dtype=torch.float64, device=dev)
                dst = bstage[key]
                if comm.i == orow:
                    dst.t().copy_(B_l[lo:lo + w, :])
                fixups.append((dst, po, w))
            works.append(comm.bcast_col(dst, orow))
        return [x for x in works if x], fixups

    bstage = {}
    pending = post(0)
    launches = 0
    for p in range(L.panels):
        nxt = post(p + 1) if p + 1 < L.panels else ([], [])
        works, fixups = pending
        for w in works:
            w.wait()
        for src, po, w in fixups:
            bbuf[p % 2][po:po + w, :].copy_(src.t())
        n = gemm(alpha, abuf[p % 2], bbuf[p % 2], C_l)
        launches += n if isinstance(n, int) else 1
        pending = nxt
    return launches


def summa_loopback(layout: Layout, A_blocks: List[torch.Tensor], B_blocks: List[torch.Tensor],
                   C_blocks: List[torch.Tensor], alpha: float = 1.0, variant="abc", level=1,
                   local_gemm: Optional[Callable] = None) -> int:
    """The same schedule with P virtual ranks in one process.

    Each "broadcast" is a copy from the owner's block, and ranks run one after another on
    one device. Nothing waits on another launch, so a single GPU can run it safely.
    Returns the GPU kernel launches of the local updates (one per update when
    `local_gemm` reports no count).
    """
    L = layout
    gemm = local_gemm or _default_local_gemm(variant, level)
    P = L.pr * L.pc
    dev = C_blocks[0].device
    abuf = torch.empty((L.b, L.m_l), dtype=torch.float64, device=dev).t()
    bbuf = torch.empty((L.n_l, L.b), dtype=torch.float64, device=dev).t()
    launches = 0
    for p in range(L.panels):
        for r in range(P):
            i, j = divmod(r, L.pc)
            for oc, lo, w, po in L.a_pieces(p):        # row-i broadcasts
                abuf[:, po:po + w].copy_(A_blocks[i * L.pc + oc][:, lo:lo + w])
            for orow, lo, w, po in L.b_pieces(p):      # column-j broadcasts
                bbuf[po:po + w, :].copy_(B_blocks[orow * L.pc + j][lo:lo + w, :])
            n = gemm(alpha, abuf, bbuf, C_blocks[r])
            launches += n if isinstance(n, int) else 1
    return launches


# ------------------------------------------------- peer-memory SUMMA (no broadcasts)
# Variants whose local update starts with a materialising operand-sum pass: that pass is
# the only reader of A and B, so it can read the owner's block in place (over NVLink on a
# real node) and the all-gather is fused into the sum pass.
DIRECT_VARIANTS = ("naive", "c")


def open_peer_blocks(A_l: torch.Tensor, B_l: torch.Tensor, group=None):
    """Map every rank's A and B blocks into this process (CUDA IPC).

    Each rank exports its blocks' IPC handles (torch.multiprocessing's CUDA tensor
    reduction: cudaIpcGetMemHandle on the allocation, plus the offset inside it); the
    handles are exchanged with all_gather_object over `group` (metadata only, a few hundred
    bytes) and opened with cudaIpcOpenMemHandle, which enables peer access on a multi-GPU
    node.  Entry r of the returned lists is rank r's block; this rank's own entry is its
    tensor.  The owners must keep A_l / B_l alive while peers use the mappings.
    """
    import torch.distributed as dist
    from torch.multiprocessing.reductions import reduce_tensor
    if not (A_l.is_cuda and B_l.is_cuda):
        raise ValueError("open_peer_blocks needs CUDA blocks")
    me = dist.get_rank(group)
    if dist.get_world_size(group) == 1:      # nothing to export (and no consumer to release it)
        return [A_l], [B_l]
    mine = (reduce_tensor(A_l), reduce_tensor(B_l))
    allh = [None] * dist.get_world_size(group)
    dist.all_gather_object(allh, mine, group=group)
    A_peers, B_peers = [], []
    for r, (ha, hb) in enumerate(allh):
        if r == me:
            A_peers.append(A_l)
            B_peers.append(B_l)
        else:
            A_peers.append(ha[0](*ha[1]))
            B_peers.append(hb[0](*hb[1]))
    return A_peers, B_peers


def summa_p2p(layout: Layout, rank: int, A_peers: List[torch.Tensor], B_peers: List[torch.Tensor],
              C_l: torch.Tensor, alpha: float = 1.0, variant="naive", level=2,
              local_gemm: Optional[Callable] = None, direct: Optional[bool] = None) -> int:
    """C_l += alpha * (A @ B)_ij with the operands read from the owners' memory.

    The same product as :func:`summa`, with no broadcast: rank (i, j) walks
    ``layout.k_pieces()`` and each rank-w update takes A columns from the block of rank
    (i, a_col) and B rows from the block of rank (b_row, j), both as strided views of the
    owners' memory (:func:`open_peer_blocks`, or local tensors for a loopback).

    * direct (default for Naive and C): the local Strassen call reads the peer views
      itself.  Its first kernels are the operand-sum passes, which read every A and B
      element once and write the sums to local HBM, so the gather over NVLink is fused
      into the pass Strassen makes anyway and no SM time goes to a collective.
    * staged (ABC, AB, classical, whose mainloop re-reads operand tiles): piece t + 1 is
      pulled into a local double buffer on a side stream while piece t's update runs.

    The caller provides the ordering across ranks: every owner's blocks must be final
    before any rank starts (device synchronize + barrier), and must not change until
    every rank has finished.  Returns the GPU launches of the local updates (one per
    update when `local_gemm` reports no count).
    """
    L = layout
    i, j = divmod(rank, L.pc)
    gemm = local_gemm or _default_local_gemm(variant, level)
    if direct is None:
        direct = variant in DIRECT_VARIANTS
    pieces = L.k_pieces()

    def views(pc):
        g0, w, ac, ao, br, bo = pc
        return A_peers[i * L.pc + ac][:, ao:ao + w], B_peers[br * L.pc + j][bo:bo + w, :]

    launches = 0
    if direct:
        for pc in pieces:
            a, b = views(pc)
            n = gemm(alpha, a, b, C_l)
            launches += n if isinstance(n, int) else 1
        return launches

    dev = C_l.device
    wmax = max(pc[1] for pc in pieces)
    abuf = [torch.empty((wmax, L.m_l), dtype=torch.float64, device=dev).t() for _ in range(2)]
    bbuf = [torch.empty((L.n_l, wmax), dtype=torch.float64, device=dev).t() for _ in range(2)]
    cuda = C_l.is_cuda
    side = torch.cuda.Stream(device=dev) if cuda else None
    main = torch.cuda.current_stream(dev) if cuda else None
    ready, free = [None, None], [None, None]

    def pull(t):
        s, w = t % 2, pieces[t][1]
        a, b = views(pieces[t])
        if not cuda:
            abuf[s][:, :w].copy_(a)
            bbuf[s][:w, :].copy_(b)
            return
        with torch.cuda.stream(side):
            if free[s] is not None:          # the update that last read buffer s is done
                side.wait_event(free[s])
            abuf[s][:, :w].copy_(a, non_blocking=True)
            bbuf[s][:w, :].copy_(b, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(side)
            ready[s] = ev

    pull(0)
    for t, pc in enumerate(pieces):
        if t + 1 < len(pieces):
            pull(t + 1)
        s, w = t % 2, pc[1]
        if cuda:
            main.wait_event(ready[s])
        n = gemm(alpha, abuf[s][:, :w], bbuf[s][:w, :], C_l)
        launches += n if isinstance(n, int) else 1
        if cuda:
            ev = torch.cuda.Event()
            ev.record(main)
            free[s] = ev
    if cuda:
        for x in abuf + bbuf:                # buffers freed on the main stream's order
            x.record_stream(side)
    return launches


# ------------------------------------------ native SUMMA (include/strassen_dist.h)
class NativeGrid:
    """One rank's handle on the library's native SUMMA (``strassen_dist_*``,
    csrc/dist.cpp): the same schedule as :func:`summa`, issued by the C++ side --
    NCCL row/column broadcasts on a communication stream, double-buffered panels,
    ``strassen_gemm_device`` as the local update.  This is what a C / C++ caller of
    the drop-in library uses; the Python class only forwards to it.
    """

    def __init__(self, ctx, handle, keep=()):
        import paper_1605_01078_b200 as S
        self._S, self._l = S, S.lib()
        self.ctx, self.ptr, self._keep = ctx, handle, keep

    # ---- schedule helpers (pure host code) ----
    @staticmethod
    def grid(nranks):
        import ctypes as C
        import paper_1605_01078_b200 as S
        pr, pc = C.c_int(), C.c_int()
        S._check(S.lib().strassen_dist_grid(int(nranks), C.byref(pr), C.byref(pc)), "dist_grid")
        return pr.value, pc.value

    @staticmethod
    def default_panel(k):
        import paper_1605_01078_b200 as S
        return S.lib().strassen_dist_default_panel(int(k))

    @staticmethod
    def panel_pieces(k, pr, pc, b, p, side):
        """Pieces of panel p as (owner, local offset, width, panel offset); side 'a' or 'b'."""
        import ctypes as C
        import paper_1605_01078_b200 as S
        out = (S.DistPiece * 64)()
        n = C.c_long()
        S._check(S.lib().strassen_dist_panel_pieces(k, pr, pc, b, p, 0 if side == "a" else 1,
                                                    out, 64, C.byref(n)), "dist_panel_pieces")
        return [(out[t].owner, out[t].local_off, out[t].width, out[t].panel_off)
                for t in range(n.value)]

    # ---- transports ----
    @staticmethod
    def unique_id() -> bytes:
        import ctypes as C
        import paper_1605_01078_b200 as S
        buf = C.create_string_buffer(128)
        S._check(S.lib().strassen_dist_unique_id(buf), "dist_unique_id")
        return buf.raw

    @classmethod
    def nccl(cls, ctx, unique_id: bytes, rank, nranks, pr, pc):
        """Collective: every rank of the job calls it with rank 0's unique id."""
        import ctypes as C
        import paper_1605_01078_b200 as S
        h = C.c_void_p()
        idbuf = C.create_string_buffer(unique_id, 128)
        S._check(S.lib().strassen_dist_create(C.byref(h), ctx.ptr, idbuf, rank, nranks, pr, pc),
                 "dist_create")
        return cls(ctx, h)

    @classmethod
    def from_torch_distributed(cls, ctx, pr, pc, group=None):
        """Joins the native NCCL job of a torch.distributed launch: rank 0 makes the
        unique id, the existing process group carries it to the other ranks."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        box = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0, group=group)
        return cls.nccl(ctx, box[0], rank, world, pr, pc)

    @classmethod
    def loopback(cls, ctx, mailbox, rank, pr, pc):
        import ctypes as C
        import paper_1605_01078_b200 as S
        h = C.c_void_p()
        S._check(S.lib().strassen_dist_create_loopback(C.byref(h), ctx.ptr, mailbox.ptr, rank,
                                                       pr, pc), "dist_create_loopback")
        return cls(ctx, h, keep=(mailbox,))

    def close(self):
        if self.ptr:
            self._l.strassen_dist_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- the multiply ----
    def gemm(self, variant, level, m, n, k, alpha, A_l, B_l, C_l, panel=0, stream=None):
        """C_l += alpha (A B)_ij for the global m x n x k product (column-major blocks)."""
        import ctypes as C
        for t in (A_l, B_l, C_l):
            if t.dim() != 2 or t.dtype != torch.float64 or (t.shape[0] > 1 and t.stride(0) != 1):
                raise ValueError("blocks must be column-major float64 matrices")
        if stream is None:
            stream = torch.cuda.current_stream(C_l.device)
        h = getattr(stream, "cuda_stream", stream)
        st = self._l.strassen_dist_gemm(
            self.ptr, C.c_void_p(h), self._S._variant(variant), int(level), m, n, k, float(alpha),
            C.c_void_p(A_l.data_ptr()), A_l.stride(1), C.c_void_p(B_l.data_ptr()), B_l.stride(1),
            C.c_void_p(C_l.data_ptr()), C_l.stride(1), int(panel))
        self._S._check(st, "strassen_dist_gemm")
        return self.last_counts()[0]

    def last_counts(self):
        import ctypes as C
        a, b = C.c_long(), C.c_long()
        self._S._check(self._l.strassen_dist_last_counts(self.ptr, C.byref(a), C.byref(b)),
                       "dist_last_counts")
        return a.value, b.value

    def position(self):
        import ctypes as C
        v = [C.c_int() for _ in range(5)]
        self._S._check(self._l.strassen_dist_position(self.ptr, *[C.byref(x) for x in v]),
                       "dist_position")
        return tuple(x.value for x in v)


class Mailbox:
    """Payload store of the native single-GPU loopback transport."""

    def __init__(self):
        import ctypes as C
        import paper_1605_01078_b200 as S
        self._l = S.lib()
        self.ptr = C.c_void_p()
        S._check(self._l.strassen_dist_mailbox_create(C.byref(self.ptr)), "mailbox_create")

    def set_replay(self, on):
        self._l.strassen_dist_mailbox_set_replay(self.ptr, int(bool(on)))

    def __del__(self):
        try:
            if self.ptr:
                self._l.strassen_dist_mailbox_destroy(self.ptr)
                self.ptr = None
        except Exception:
            pass


def summa_native_loopback(layout: Layout, A_blocks, B_blocks, C_blocks, alpha=1.0,
                          variant="abc", level=1) -> int:
    """The native schedule for every rank of the grid on ONE GPU: a record pass (roots'
    payloads kept, C restored afterwards) and a replay pass (every broadcast delivers the
    recorded payload).  Ranks run one after another; nothing waits on another launch."""
    import paper_1605_01078_b200 as S
    L = layout
    P = L.pr * L.pc
    mb = Mailbox()
    ctx = S.Ctx()
    grids = [NativeGrid.loopback(ctx, mb, r, L.pr, L.pc) for r in range(P)]
    saved = [c.clone() for c in C_blocks]
    launches = 0
    for replay in (False, True):
        mb.set_replay(replay)
        for r in range(P):
            if replay:
                C_blocks[r].copy_(saved[r])
            n = grids[r].gemm(variant, level, L.m, L.n, L.k, alpha, A_blocks[r], B_blocks[r],
                              C_blocks[r], panel=L.b)
            if replay:
                launches += n
    torch.cuda.synchronize()
    for g in grids:
        g.close()
    return launches
