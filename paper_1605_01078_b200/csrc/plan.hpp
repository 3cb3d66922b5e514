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

}  // namespace sb200
