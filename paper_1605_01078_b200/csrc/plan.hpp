// Launch planning shared by the engine (engine.cpp plan_fused) and the B200
// cost model (accounting.cpp b200_predict_seconds), so the model predicts the
// launches the engine actually makes.
#pragma once
#include <cmath>

namespace sb200 {

// Split mode (one CTA per tile x product x k-chunk, partials + one stream
// pass): the k-chunk count minimising
//   waves(CTAs) x (chunk k-tiles x t_k + t_cta) + stream pass (bandwidth or
//   the latency of its per-thread chain of partial loads),
// where a 16-k tile costs t_k = 2.1 us x term_factor of DMMA work (4096 cycles
// at 1.965 GHz; term_factor > 1 for fused operand sums) and t_cta ~3 us covers
// a CTA's prologue, pipeline fill and epilogue.  q_elems = qm * qn (one
// product's partial).  Returns the chunk count; *per = k-tiles per chunk.
inline int choose_ksplit(long ntiles, long nprod, long ktiles, long sms, double q_elems,
                         double term_factor, long* per_out) {
    const double t_k = 2.1e-6 * term_factor, t_cta = 3.0e-6, bw = 5.0e12;
    double best = 1e300;
    int best_ks = 1;
    long best_per = ktiles;
    for (long ks = 1; ks <= 64 && ks <= ktiles; ++ks) {
        const long per = (ktiles + ks - 1) / ks;
        const long ks2 = (ktiles + per - 1) / per;
        if (ks2 != ks) continue;  // same chunking as a smaller ks
        const double ctas = static_cast<double>(ntiles) * nprod * ks2;
        const double waves = std::ceil(ctas / static_cast<double>(sms));
        // stream pass: bandwidth, or at small sizes the chain of nprod * ks dependent
        // partial loads per thread (~0.7 us each; 1024^3 Naive L2 measured 68 us at ks = 2)
        const double t_stream = std::fmax(8.0 * q_elems * nprod * ks2 / bw, nprod * ks2 * 0.7e-6);
        const double t = waves * (per * t_k + t_cta) + t_stream;
        if (t < best * 0.995) {  // prefer fewer chunks on near-ties
            best = t;
            best_ks = static_cast<int>(ks2);
            best_per = per;
        }
    }
    if (per_out) *per_out = best_per;
    return best_ks;
}

// Dynamic peeling (engine.cpp run_device): the core extent of a dimension d at level L
// (S = 2^L) -- the multiple of S below d, or, where d exceeds a whole number of quadrant
// tiles by at most the fringe kernels' width w, the multiple of S x tile below it.
inline long peel_core(long d, long S, long tile, long w) {
    const long rem = d % (S * tile);
    if (rem > 0 && rem <= w && d > rem) return d - rem;
    return d & ~(S - 1);
}

// Peeling pays when the padded tile steps it removes (work counts 128 x 128 x 16 steps of
// one product; nprod = 7^L products; 2.1 us per step on one of `sms` SMs) outweigh the
// fringe updates: their launches (~40 us) and their HBM passes (measured 2-5 TB/s;
// profiles/r02_tile_peel_ab.log: 2052^3 classical loses, 4100^3 gains).
inline bool peel_pays(long work_full, long work_core, long nprod, long sms, double fringe_bytes) {
    return static_cast<double>(work_full - work_core) * nprod * 2.1e-6 / sms >
           40e-6 + fringe_bytes / 2.0e12;
}
// HBM bytes of the three fringe updates of an m x n x k problem peeled to me x ne x ke
inline double fringe_bytes(long m, long n, long k, long me, long ne, long ke) {
    double b = 0.0;
    if (ke < k) b += 16.0 * static_cast<double>(me) * ne;
    if (me < m) b += 8.0 * static_cast<double>(k) * n;
    if (ne < n) b += 8.0 * static_cast<double>(me) * k;
    return b;
}

// Classical launches of four or more waves of tile owners: the last, partial wave
// leaves SMs idle (3840^3: 900 tiles on 148 SMs run as 7 waves for 6.08 waves of work).
// Hybrid: the first tile columns as whole waves of tile owners, the last `cols` tile
// columns (the "tail") as stream-K pieces balanced over every SM.  Returns the tail's
// tile columns (0 = none: the plain tile-owner grid is within 3% of it) and the
// predicted time of the choice.
struct TailPlan {
    long cols = 0;
    double t = 0.0;
};
inline TailPlan choose_tail(long tiles_m, long tiles_n, long ktiles, long sms) {
    const double t_k = 2.1e-6, t_cta = 3e-6;
    const double t_tile = static_cast<double>(ktiles) * t_k + t_cta;
    TailPlan best;
    best.t = std::ceil(static_cast<double>(tiles_m) * tiles_n / sms) * t_tile;
    const double t_plain = best.t;
    for (long ct = 1; ct < tiles_n; ++ct) {
        const double body = static_cast<double>(tiles_m) * (tiles_n - ct);
        const double tail = static_cast<double>(tiles_m) * ct;
        if (tail > 2.0 * sms) break;  // (a tail of up to two waves of tiles)
        const double len = std::ceil(tail * ktiles / sms);
        // stream-K pieces: 2.22 us per k-step and ~30 us of fixup and launch
        // (profiles/r02_streamk_wide_ab.log)
        const double t = std::ceil(body / sms) * t_tile + len * 2.22e-6 + 30e-6;
        if (t < best.t) {
            best.t = t;
            best.cols = ct;
        }
    }
    if (best.t > 0.97 * t_plain) {
        best.cols = 0;
        best.t = t_plain;
    }
    return best;
}

}  // namespace sb200
