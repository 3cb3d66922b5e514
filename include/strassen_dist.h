/*
 * strassen_dist.h -- native distributed entry points of libstrassen_b200.so:
 * SUMMA on a 2-D process grid with the local Strassen call as the rank-b update.
 *
 * The reference has no distributed API.  What it has is the single-process
 * rank-b schedule of its bench library (proj/tools/bench_lib.cpp:56-71:
 * C += sum_p A[:, p0:p0+b] B[p0:p0+b, :] through repeated strassen_gemm), which
 * is what the paper's distributed experiment runs on every node under SUMMA
 * (PAPER.md:140-195).  These functions are that experiment for a C / C++ caller
 * of the drop-in library: one process (or thread) per GPU, each owning one block
 * of A, B and C, NCCL broadcasts along process rows and columns, and
 * strassen_gemm_device as the local update.
 *
 * Distribution.  Rank r of a pr x pc grid sits at
 * (i, j) = (r / pc, r % pc) and owns, all column-major:
 *   A_ij = A[i*m/pr : (i+1)*m/pr, j*k/pc : (j+1)*k/pc]    lda >= m/pr
 *   B_ij = B[i*k/pr : (i+1)*k/pr, j*n/pc : (j+1)*n/pc]    ldb >= k/pr
 *   C_ij = C[i*m/pr : (i+1)*m/pr, j*n/pc : (j+1)*n/pc]    ldc >= m/pr
 * One exchange step per k-panel of width b: the owners of A's panel broadcast
 * their pieces along the process row, the owners of B's panel along the process
 * column (a panel straddling owners is assembled from one broadcast per owning
 * piece); then C_ij += alpha * A_panel * B_panel locally.  The broadcasts of
 * panel p + 1 run on a communication stream while panel p's update runs.
 *
 * There is no CPU fallback: strassen_dist_gemm needs a CUDA device.  The
 * schedule functions (grid, panel pieces) are pure host code.
 */
#ifndef STRASSEN_B200_DIST_H
#define STRASSEN_B200_DIST_H

#include <stddef.h>

#include "strassen.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct strassen_dist strassen_dist;

/* ---- schedule (host only; the Python layer's Layout, summa.py) ------------- */

/* Most-square pr x pc grid with pr <= pc: 1 -> 1x1, 2 -> 1x2, 4 -> 2x2, 8 -> 2x4. */
strassen_status strassen_dist_grid(int nranks, int* pr_out, int* pc_out);

/* Default panel width for depth k: k halved while above 8192 (bounds the two
 * double-buffered panels; profiles/r01_sweep_rankk.csv). */
long strassen_dist_default_panel(long k);

/* One piece of a k-panel: the process column (A) or process row (B) that owns
 * it, the offset inside that owner's block, its width, and its offset inside
 * the panel. */
typedef struct strassen_dist_piece {
    int owner;
    long local_off;
    long width;
    long panel_off;
} strassen_dist_piece;

/* Pieces of panel p (global k range [p*b, (p+1)*b)) cut at owner boundaries.
 * side 0 = A (owners are process columns, k/pc columns each), side 1 = B
 * (owners are process rows, k/pr rows each).  Writes at most cap pieces to out
 * and returns the piece count in *count_out.  PARAM when k does not divide the
 * grid, b does not divide k, or p is out of range. */
strassen_status strassen_dist_panel_pieces(long k, int pr, int pc, long b, long p, int side,
                                           strassen_dist_piece* out, long cap, long* count_out);

/* ---- transports ------------------------------------------------------------ */

/* NCCL unique id (128 bytes, ncclGetUniqueId): made by one rank and handed to
 * every rank by the caller's own means (MPI_Bcast, a file, a socket). */
#define STRASSEN_DIST_ID_BYTES 128
strassen_status strassen_dist_unique_id(void* id_out);

/* Joins the NCCL job (ncclCommInitRank on the current CUDA device) and splits
 * the row and column communicators (ncclCommSplit, colour = grid row / column).
 * nranks must equal pr * pc.  Collective: every rank calls it.  The ctx is
 * borrowed and must outlive the handle; it runs the local updates.  NCCL is
 * resolved at run time (libnccl.so.2); when it is missing: STRASSEN_ERR_DEVICE. */
strassen_status strassen_dist_create(strassen_dist** out, strassen_ctx* ctx, const void* id,
                                     int rank, int nranks, int pr, int pc);

/* The same on a communicator the caller already has (ncclComm_t as void*; not
 * destroyed with the handle). */
strassen_status strassen_dist_create_from_comm(strassen_dist** out, strassen_ctx* ctx,
                                               void* nccl_comm, int pr, int pc);

/* A caller-supplied transport (e.g. CUDA-aware MPI_Bcast).  bcast must enqueue,
 * on CUDA stream `stream`, a broadcast of `count` doubles from grid position
 * `root` of this rank's process row (axis 0: root is a process column) or
 * process column (axis 1: root is a process row); the root's data is at `send`,
 * every rank (the root too) receives at `recv`; send == recv is allowed.
 * Non-zero return = failure (STRASSEN_ERR_DEVICE). */
typedef struct strassen_dist_transport {
    int (*bcast)(void* user, int axis, const double* send, double* recv, size_t count, int root,
                 void* stream);
    void (*destroy)(void* user); /* may be NULL */
    void* user;
} strassen_dist_transport;

strassen_status strassen_dist_create_custom(strassen_dist** out, strassen_ctx* ctx,
                                            const strassen_dist_transport* transport, int rank,
                                            int pr, int pc);

/* Single-GPU loopback transport: P virtual ranks of ONE process run their
 * strassen_dist_gemm calls one after another, twice.  In the record pass every
 * root's payload is kept in the mailbox (receivers get nothing); in the replay
 * pass every broadcast delivers the recorded payload.  Nothing waits on another
 * launch, so one GPU runs the whole grid's data path with the real kernels.
 * (The counterpart of summa.summa_loopback for the native schedule.) */
typedef struct strassen_dist_mailbox strassen_dist_mailbox;
strassen_status strassen_dist_mailbox_create(strassen_dist_mailbox** out);
void strassen_dist_mailbox_destroy(strassen_dist_mailbox* mb);
strassen_status strassen_dist_mailbox_set_replay(strassen_dist_mailbox* mb, int replay);
strassen_status strassen_dist_create_loopback(strassen_dist** out, strassen_ctx* ctx,
                                              strassen_dist_mailbox* mb, int rank, int pr, int pc);

void strassen_dist_destroy(strassen_dist* d);

/* ---- the distributed multiply ---------------------------------------------- */

/* C_ij += alpha * (A B)_ij for the GLOBAL m x n x k product; a, b, c are this
 * rank's blocks in device memory (column-major, see above).  panel = 0 picks
 * strassen_dist_default_panel(k).  Collective over the grid; asynchronous on
 * `stream` (cudaStream_t as void*, NULL = legacy default stream): C_ij is
 * updated in stream order, and A_ij / B_ij may be changed by work enqueued on
 * `stream` after the call returns.
 * Validation: NULL -> ERR_NULL; variant / level as strassen_gemm; m % pr, n % pc,
 * k % pr, k % pc, k % panel != 0, or a leading dimension below the block's rows
 * -> ERR_PARAM; host pointers -> ERR_PARAM. */
strassen_status strassen_dist_gemm(strassen_dist* d, void* stream, strassen_variant variant,
                                   int level, long m, long n, long k, double alpha,
                                   const double* a, long lda, const double* b, long ldb,
                                   double* c, long ldc, long panel);

/* Kernels launched by the local updates of the last strassen_dist_gemm, and the
 * number of exchange steps (panels) it ran. */
strassen_status strassen_dist_last_counts(const strassen_dist* d, long* launches_out,
                                          long* panels_out);

/* Grid position of this handle. */
strassen_status strassen_dist_position(const strassen_dist* d, int* rank, int* pr, int* pc,
                                       int* row, int* col);

#ifdef __cplusplus
}
#endif

#endif /* STRASSEN_B200_DIST_H */
