// Device-side parameter blocks and launchers shared by the host engine
// (engine.cpp) and the sm_100a kernels (kernels.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace sb200 {

// ---- fused Strassen tile kernel (mm_kernel) -------------------------------
constexpr int kBM = 128;            // CTA tile rows (logical quadrant rows)
constexpr int kBN = 128;            // CTA tile cols
constexpr int kBK = 16;             // k per pipeline step
constexpr int kMaxQuad = 16;        // 2^L x 2^L quadrants, L <= 2
constexpr int kMaxMaps = 64;        // tensor maps per side: 16 quadrants + materialised sums
constexpr int kMaxProducts = 49;    // 7^L
constexpr int kMaxTerms = 4;        // operand terms / destinations per product at L <= 2
constexpr int kConsumerWarps = 8;   // 2 warpgroups; 2 (m) x 4 (n) warps of 64 x 32
constexpr int kThreads = 128 + kConsumerWarps * 32;  // 384: + TMA warpgroup (1 active warp)
constexpr int kSlotBytes = kBM * kBK * 8;            // one 128x16 fp64 operand tile (16 KB)
constexpr int kRawSlots = 14;                        // TMA ring of operand-term tiles (224 KB)
constexpr int kProducerRegs = 24;                    // setmaxnreg split
constexpr int kConsumerRegs = 240;
// setmaxnreg moves registers inside the CTA's launch allocation (384 threads x
// 168 = 64512): the DMMA warps' increase must be covered by the producer
// warpgroup's release, or setmaxnreg.inc waits forever.
static_assert(kProducerRegs * 128 + kConsumerRegs * kConsumerWarps * 32 <= kThreads * 168,
              "setmaxnreg split exceeds the CTA register allocation");
// ring + alignment slack (up to 1023 bytes) + ring and unit-queue barriers
constexpr int kMMSmemBytes = kRawSlots * kSlotBytes + 1024 + 512;
static_assert(kMMSmemBytes <= 227 * 1024, "shared memory budget");
// persistent single-term launches with the deferred bulk epilogue: a 5-slot
// ring (2.5 k-steps of (1, 1) products ahead) and a separate 130 KB stage of
// one C tile (128 columns x 1040 B: the 16-byte skew spreads banks)
constexpr int kSepRing = 5;
// the same for fused-sum programs of at most 2 + 2 terms (4 term tiles per k-step):
// 6 slots, the most that fit beside the stage
constexpr int kSepRing2 = 6;
constexpr int mm_sep_smem_bytes(int ring) { return ring * kSlotBytes + 1024 + 1024 + kBM * kBN * 8; }
// (the stage holds one C tile as 8 swizzled boxes of 16 rows x 128 columns,
// 1024-byte aligned after the ring's barriers)
constexpr int kStageBytes = kBM * kBN * 8;
constexpr int kMMSepSmemBytes = kSepRing * kSlotBytes + 1024 + 1024 + kStageBytes;
static_assert(kMMSepSmemBytes <= 227 * 1024, "shared memory budget (separate stage)");
static_assert(mm_sep_smem_bytes(kSepRing2) <= 227 * 1024, "shared memory budget (fused, separate stage)");
// Narrow tiles (MMParams::narrow, small problems): 128 x 64 CTA tiles, one DMMA
// warpgroup (2 x 2 warps of 64 x 32) + the TMA warpgroup, TWO CTAs per SM, so one
// CTA's prologue, fixup and epilogue overlap the other's mainloop.  Per CTA: half
// the SM's registers (256 threads x 128 at launch; setmaxnreg 24 / 232) and a
// 6-slot ring (a B term tile uses half a slot).
constexpr int kNarrowBN = 64;
constexpr int kNarrowConsumerWarps = 4;
constexpr int kNarrowThreads = 128 + kNarrowConsumerWarps * 32;  // 256
constexpr int kNarrowConsumerRegs = 232;
static_assert(kProducerRegs * 128 + kNarrowConsumerRegs * kNarrowConsumerWarps * 32 <=
                  kNarrowThreads * 128,
              "narrow setmaxnreg split exceeds half the SM's registers");
constexpr int kNarrowRing = 6;
constexpr int kNarrowSmemBytes = kNarrowRing * kSlotBytes + 1024 + 512;
static_assert(2 * (kNarrowSmemBytes + 1024) <= 228 * 1024, "two narrow CTAs per SM");
// dynamic unit hand-out queue (MMParams::unit_counter): depth, after the ring barriers
constexpr int kUnitQueue = 4;
static_assert(2 * kSepRing * 8 + 2 * kUnitQueue * 8 + kUnitQueue * 4 <= 1024,
              "ring and queue barriers fit before the stage");
static_assert(2 * kRawSlots * 8 + 2 * kUnitQueue * 8 + kUnitQueue * 4 <= 1024,
              "ring and queue barriers fit in the reserved kilobyte");

// One Strassen product M_p = (sum_u as_u A_{aq_u}) (sum_u bs_u B_{bq_u});
// destinations C_{cq_u} += alpha * cs_u * M_p.
struct ProductDesc {
    int8_t na, nb, nc;
    int8_t half;  // stream 8-k half tiles, two per ring slot (4 + 4-term products)
    int8_t aq[kMaxTerms], as[kMaxTerms];
    int8_t bq[kMaxTerms], bs[kMaxTerms];
    int8_t cq[kMaxTerms], cs[kMaxTerms];
};

enum EpilogueMode : int {
    kEpiRMW = 0,    // C_q += alpha * gamma * M (ABC, DGEMM)
    kEpiStore = 1,  // M_p := M into product temporaries (AB, Naive)
};

struct alignas(64) MMParams {
    CUtensorMap tmA[kMaxMaps];  // A operands: dims (rows, cols), box 16 x 16, swizzle 128B
    CUtensorMap tmB[kMaxMaps];  // B operands: dims (k rows, n cols), box 16 x 128, swizzle 128B
    // half-k maps of the 16 quadrants for ProductDesc::half products:
    // A box 16 x 8 (128B swizzle), B box 8 x 128 (64B swizzle)
    CUtensorMap tmAh[kMaxQuad];
    CUtensorMap tmBh[kMaxQuad];
    // C quadrants (c_tma): dims (rows, cols), box 16 x 128, swizzle 128B -- the
    // bulk-reduction epilogue's TMA reduce-add targets (clipped by the map)
    CUtensorMap tmC[kMaxQuad];
    ProductDesc prod[kMaxProducts];
    double* cptr[kMaxQuad];     // C quadrant views (clipped)
    int crows[kMaxQuad];
    int ccols[kMaxQuad];
    long long rs_c, cs_c;
    double* mbase;              // kEpiStore: M_p = mbase + p * mstride, col-major, ld = ldm
    long long mstride;
    long long ldm;
    double alpha;
    int nprod;
    int qm, qn, qk;             // logical quadrant extents
    int tiles_m, tiles_n, ktiles;
    int mode;
    int group_m;                // tile rasterisation group height
    int tm0, tn0;               // first tile row / column (windows of the host pipeline)
    int c_vec;                  // C column-major, even ldc, 16-byte aligned quadrants
    // split mode (few output tiles): blockIdx -> (tile, product, k-chunk); each
    // CTA stores its partial product to M_{p*ksplit+s} (kEpiStore)
    int split;
    int ksplit, kt_per_split;
    // ticketed fused epilogue (kEpiRMW): CTA (tile, p) applies its C updates once
    // tickets[tile] == p, then sets it to p + 1, so every C tile receives the
    // products in table order (deterministic).  (Per-(tile, quadrant) tickets were
    // measured ~3% slower for short fused products: profiles/r02_shortk6.log.)
    int* tickets;
    int ticket_ld;              // tickets row stride (tile columns of the whole call)
    // k-split fused epilogue (split grid, ksplit > 1, kEpiRMW): every CTA of
    // (tile, product) stores its partial to M_{p,s}; the last to arrive
    // (counter arrive[tile * nprod + p]) sums the partials in s order and does
    // the ticketed read-modify-write -- no separate stream pass
    int* arrive;
    // fused epilogue through TMA bulk f64 reductions for CTAs of at most this
    // many k-tiles (short products, where the register read-modify-write would
    // be a large share of the CTA); 0 = never
    int bulk_max_kt;
    // persistent launch: at most this many CTAs (one per SM), each walking
    // units blockIdx.x + i * gridDim.x; 0 = one CTA per unit
    int grid_cap;
    // ticketed grid (split, ksplit = 1): units in groups of this many tiles,
    // product-major inside a group, so a group's C tiles stay L2-resident across
    // its 7^L ordered updates; 0 = product-major over all tiles
    int unit_group;
    // persistent single-term launch whose bulk-reduction epilogues use a separate
    // stage and collect their completion one unit later (kSepRing ring slots)
    int sep_stage;
    // sep_stage: collect a unit's reductions (and release its ticket) only at the
    // CTA's next epilogue.  Safe for throughput when a tile's next product is at
    // least two grid-widths of units away (else it would wait a whole unit)
    int sep_defer;
    int c_tma;  // tmC valid: bulk epilogue through tensor reduce-adds (partial tiles too)
    // stream-K (single-product programs with under two waves of tiles): persistent
    // CTA c covers k-steps [c * sk_len, (c + 1) * sk_len) of the flattened (tile,
    // k-step) space, at most sk_maxp pieces; partial pieces go through the k-split
    // fixup (ksplit = partial slots per tile, arrive counters per tile)
    int streamk, sk_len, sk_maxp;
    // stream-K over (tile, product, k-step) for store-mode programs (kEpiStore, few
    // tiles): a (tile, product) cut into pieces stores them as partials at
    // mbase + part_off + (p * ksplit + piece) * mstride; the last piece to arrive
    // sums them in piece order and stores M_p at mbase + p * mstride (ksplit = 1 for
    // the stream pass).  part_off = 0 and sk_store = 0 elsewhere (the RMW k-split
    // fixup keeps its partials at mbase).
    int sk_store;
    long long part_off;
    // Cooperative fixup (k-chunk grids whose CTAs are all resident with one unit each;
    // stream-K launches too under STRASSEN_B200_COOP_SK, off by default: no gain
    // measured): the pieces of a (tile, product) that are their CTA's last unit
    // ("participants") share the fixup instead of one owner doing all of it.  Every piece
    // stores its partial and arrives; after its unit loop -- where the accumulators and
    // the ring state are dead, so the code costs the k-loops no registers -- a participant
    // waits until every piece has arrived, sums the partials of the 64 x 8 fragment blocks
    // b = 4 warp + nf with b % participants == its index (ascending piece order, the
    // single-owner fixup's arithmetic, bit for bit) and applies the epilogue to them.  A
    // piece with units after it (the tail piece at the start of a stream-K range) only
    // stores its partial and arrives.
    int coop_fixup;
    // A-heavy products (more A than B terms) in one-CTA-per-unit launches run the
    // 4 x 2 warp layout (kernels.cu product_kloop1)
    int a_heavy_layout;
    // persistent launches (not stream-K): units beyond the first wave are handed out
    // by this counter (zeroed before the launch), so a CTA that starts late -- an SM
    // held by another kernel, e.g. a co-scheduled NCCL broadcast -- simply takes fewer
    // units instead of delaying a fixed list; units are still taken in increasing
    // order, so ticket waits (which point at smaller units) cannot deadlock
    int* unit_counter;
    // Product groups (ticketed fused-epilogue grid): a unit is (tile, group j) covering
    // products [pair_lo[j], pair_lo[j + 1]) -- one to three products whose destination
    // sets overlap (the host orders them adjacently).  The first products' accumulators
    // are parked in tensor memory (tcgen05.st) while the last one's mainloop runs; the
    // epilogue then applies alpha (g1 M1 + g2 M2 + g3 M3) to each destination with ONE
    // update, so a shared destination is read and written once instead of two or three
    // times.  Tickets count groups.  0 = one product per unit.
    // SB200_TRACE builds only (libstrassen_b200_trace.so): per-CTA %globaltimer events,
    // 32 slots per CTA -- 0 entry, 31 exit, 1 + 2i / 2 + 2i unit i's start / epilogue start
    unsigned long long* trace;
    int pair_mode;
    int npairs;
    int8_t pair_lo[kMaxProducts + 1];
    // narrow tiles (kNarrowBN columns, two CTAs per SM): tiles_n / tn0 count 64-column
    // tiles, tmB boxes are 16 x 64, register epilogues only (no c_tma, groups or half tiles)
    int narrow;
};

cudaError_t launch_mm(const MMParams& p, cudaStream_t s);

// ---- layout normalisation (TMA staging) -----------------------------------
// dst(rowmap(i), j) = src(i, j), src element (i, j) at src[i*rs + j*cs];
// rowmap(i) = (i / q) * q_al + i % q (quadrant rows placed at aligned
// offsets); dst column-major with leading dimension ld.
cudaError_t launch_repack(const double* src, long long rs, long long cs, long rows, long cols,
                          double* dst, long long ld, long q, long q_al, cudaStream_t s);

// ---- C variant: materialise many operand sums in one launch ----------------
// job z: dst_z(i, j) = sum_u c_u X_{z,u}(i, j) over a rows x cols logical extent,
// zero outside each term's clipped view; sources column-major (rs = 1).
constexpr int kMaxSumJobs = 98;
struct SumTerm {
    const double* x;
    int rows, cols;
    long long ld;
    int coeff;
};
struct SumBatchParams {
    SumTerm t[kMaxSumJobs][kMaxTerms];
    double* dst[kMaxSumJobs];
    int nterms[kMaxSumJobs];
    int njobs;
    long long rows, cols, ld;
    long long r0, c0;  // first row / column computed (rows, cols = one past the last)
};
cudaError_t launch_sum_batch(const SumBatchParams& p, cudaStream_t s);

// ---- AB / Naive: stream products into C quadrants -------------------------
constexpr int kMaxFanIn = 16;
struct StreamParams {
    double* cptr[kMaxQuad];
    int crows[kMaxQuad], ccols[kMaxQuad];
    int nsrc[kMaxQuad];
    int8_t src_prod[kMaxQuad][kMaxFanIn];
    int8_t src_coeff[kMaxQuad][kMaxFanIn];
    long long rs_c, cs_c;
    const double* mbase;
    long long mstride, ldm;
    double alpha;
    int nquad;
    int qm, qn;
    int ksplit;  // M_p = sum_{s < ksplit} mbase[(p*ksplit + s) * mstride], s ascending
    int r0, r1, c0, c1;  // quadrant window: rows [r0, r1), columns [c0, c1)
    int c_vec;           // C column-major, even ldc, 16-byte aligned quadrants
};
cudaError_t launch_stream_update(const StreamParams& p, cudaStream_t s);

// ---- fringe updates of dynamic peeling (fringe.cu) ---------------------------
// one dimension of at most fringe_max_width(): streaming kernels, the long operand read
// once; k-chunk partials in `part` (fringe_partial_bytes) added in ascending order
int fringe_max_width();
size_t fringe_partial_bytes(long long_len, int thin, long K);
// k-chunk partials of A (M x K) B (K x nf) / of A (mf x K) B (K x N), then
// C += alpha * (their sum in ascending chunk order)
cudaError_t launch_fringe_n(const double* A, long long rs_a, long long cs_a, const double* B,
                            long long rs_b, long long cs_b, long M, int nf, long K, double* part,
                            int* nkc_out, cudaStream_t s);
cudaError_t launch_fringe_m(const double* A, long long rs_a, long long cs_a, const double* B,
                            long long rs_b, long long cs_b, int mf, long N, long K, double* part,
                            int* nkc_out, cudaStream_t s);
cudaError_t launch_fringe_reduce(const double* part, int nkc, int thin, long len, double alpha,
                                 double* C, long long sl, long long st, cudaStream_t s);
// C (M x N) += alpha A (M x kf) B (kf x N)
cudaError_t launch_fringe_k(const double* A, long long rs_a, long long cs_a, const double* B,
                            long long rs_b, long long cs_b, double* C, long long rs_c,
                            long long cs_c, long M, long N, int kf, double alpha, cudaStream_t s);

// ---- beta pre-scale for the dgemm shim -------------------------------------
cudaError_t launch_scale(double* c, long rows, long cols, long long rs, long long cs, double beta,
                         cudaStream_t s);

}  // namespace sb200
