// Instrumentation counters and the analytical model of the reference, kept for
// ABI parity (strassen_ctx_get_counters, strassen_model_predict, ...).
//
// Counters: the reference increments atomics inside its CPU packing, micro-
// kernel and streaming loops (counters.hpp:8-49, blocking.cpp:33-37 / 61-65,
// kernel.cpp:42-47 / 71-75, variants.cpp:67-108).  The GPU path has no such
// loops, so the same numbers are produced here analytically by walking the
// reference's loop structure (jc / pc / ic / ir) for the ctx blocking without
// touching data -- O((n/nc)(k/kc)(m/mr)) integer work, only when enabled.
//
// Model: the paper's T = T_a + T_m (model.cpp:8-134) with the reference's
// coefficient table (including its 154/462/194 level-2 figures).
#include "accounting.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>

#include "plan.hpp"
#include "table.hpp"

namespace sb200 {
namespace {

long ceil_div(long a, long b) { return (a + b - 1) / b; }
long clampl(long v, long lo, long hi) { return std::max(lo, std::min(hi, v)); }

struct Ext {
    long rows, cols;
    bool empty() const { return rows <= 0 || cols <= 0; }
};

bool all_empty(const std::vector<Ext>& v) {
    for (const Ext& e : v)
        if (!e.empty()) return false;
    return true;
}

// gemm_five_loop (blocking.cpp:82-131) counting only.
void five_loop(long lm, long ln, long lk, const std::vector<Ext>& a, const std::vector<Ext>& b,
               const std::vector<Ext>& d, const strassen_blocking& bp,
               strassen_counter_values& c) {
    if (lm <= 0 || ln <= 0 || lk <= 0) return;
    if (all_empty(a) || all_empty(b) || all_empty(d)) return;
    for (long jc = 0; jc < ln; jc += bp.nc) {
        const long n_c = std::min(bp.nc, ln - jc);
        for (long pc = 0; pc < lk; pc += bp.kc) {
            const long k_c = std::min(bp.kc, lk - pc);
            c.pack_b_calls += 1;
            for (size_t t = 0; t < b.size(); ++t) {
                const long depth = clampl(b[t].rows - pc, 0, k_c);
                const long cols = clampl(b[t].cols - jc, 0, n_c);
                c.pack_b_elems += cols * depth;
                if (t > 0) c.pack_b_add_flops += 2 * cols * depth;
            }
            for (long ic = 0; ic < lm; ic += bp.mc) {
                const long m_c = std::min(bp.mc, lm - ic);
                c.pack_a_calls += 1;
                for (size_t t = 0; t < a.size(); ++t) {
                    const long rows = clampl(a[t].rows - ic, 0, m_c);
                    const long depth = clampl(a[t].cols - pc, 0, k_c);
                    c.pack_a_elems += rows * depth;
                    if (t > 0) c.pack_a_add_flops += 2 * rows * depth;
                }
                // macro_kernel (kernel.cpp:79-102): tiles in range of any dest
                const long m_tiles = ceil_div(m_c, bp.mr), n_tiles = ceil_div(n_c, bp.nr);
                for (long ir = 0; ir < m_tiles; ++ir) {
                    const long tr = ic + ir * bp.mr;
                    long cmax = -1;
                    for (const Ext& e : d)
                        if (tr < e.rows) cmax = std::max(cmax, e.cols);
                    if (cmax <= jc) continue;
                    const long n_in = std::min(n_tiles, ceil_div(cmax - jc, bp.nr));
                    const long in_rows = std::min(bp.mr, m_c - ir * bp.mr);
                    const long width = std::min(n_in * bp.nr, n_c);
                    c.kernel_calls += n_in;
                    c.kernel_fma_flops += 2 * k_c * std::min(in_rows, bp.mr) * width;
                    for (const Ext& e : d) {
                        if (tr >= e.rows) continue;
                        const long rw = std::min(bp.mr, e.rows - tr);
                        const long cw = std::max(0L, std::min(e.cols, jc + n_in * bp.nr) - jc);
                        c.kernel_c_elems += 2 * rw * cw;
                        c.kernel_update_flops += 2 * rw * cw;
                    }
                }
            }
        }
    }
}

std::vector<Ext> partition(long rows, long cols, int level, long& qr, long& qc) {
    const long side = 1L << level;
    qr = ceil_div(rows, side);
    qc = ceil_div(cols, side);
    std::vector<Ext> v(static_cast<size_t>(side * side));
    for (long I = 0; I < side; ++I)
        for (long J = 0; J < side; ++J)
            v[I * side + J] = {clampl(rows - I * qr, 0, qr), clampl(cols - J * qc, 0, qc)};
    return v;
}

std::vector<Ext> pick(const Terms& t, const std::vector<Ext>& g) {
    std::vector<Ext> out;
    for (const auto& x : t) out.push_back(g[x.first]);
    return out;
}

// materialize_sum (variants.cpp:53-96) pass accounting.
void materialize(size_t nterms, long rows, long cols, int64_t& passes, int64_t& elems,
                 int64_t& flops) {
    const int64_t rc = static_cast<int64_t>(rows) * cols;
    if (nterms == 1) {
        passes += 2;
        elems += 2 * rc;
    } else {
        passes += 3;
        elems += 3 * rc;
        flops += 2 * rc;
    }
    for (size_t s = 2; s < nterms; ++s) {
        passes += 3;
        elems += 3 * rc;
        flops += 2 * rc;
    }
}

}  // namespace

void count_call(strassen_variant variant, int level, long m, long n, long k,
                const strassen_blocking& bp, strassen_counter_values& c) {
    if (variant == STRASSEN_DGEMM || level == 0) {
        five_loop(m, n, k, {{m, k}}, {{k, n}}, {{m, n}}, bp, c);
        return;
    }
    long qm, qk, qk2, qn, qm2, qn2;
    const std::vector<Ext> ga = partition(m, k, level, qm, qk);
    const std::vector<Ext> gb = partition(k, n, level, qk2, qn);
    const std::vector<Ext> gc = partition(m, n, level, qm2, qn2);
    for (const Product& e : (level == 3 ? program_level3() : program_for_level(level)).products) {
        const std::vector<Ext> a = pick(e.a, ga), b = pick(e.b, gb), d = pick(e.c, gc);
        if (all_empty(a) || all_empty(b) || all_empty(d)) continue;
        if (variant == STRASSEN_ABC) {
            five_loop(qm, qn, qk, a, b, d, bp, c);
            continue;
        }
        if (variant == STRASSEN_C) {  // B200 addition: Naive's sums, ABC's fused C
            if (e.a.size() > 1)
                materialize(e.a.size(), qm, qk, c.a_plus_passes, c.a_plus_elems, c.a_plus_flops);
            if (e.b.size() > 1)
                materialize(e.b.size(), qk, qn, c.b_plus_passes, c.b_plus_elems, c.b_plus_flops);
            five_loop(qm, qn, qk, {e.a.size() > 1 ? Ext{qm, qk} : a[0]},
                      {e.b.size() > 1 ? Ext{qk, qn} : b[0]}, d, bp, c);
            continue;
        }
        if (variant == STRASSEN_AB) {
            five_loop(qm, qn, qk, a, b, {{qm, qn}}, bp, c);
        } else {
            materialize(e.a.size(), qm, qk, c.a_plus_passes, c.a_plus_elems, c.a_plus_flops);
            materialize(e.b.size(), qk, qn, c.b_plus_passes, c.b_plus_elems, c.b_plus_flops);
            five_loop(qm, qn, qk, {{qm, qk}}, {{qk, qn}}, {{qm, qn}}, bp, c);
        }
        for (const Ext& x : d) {
            if (x.empty()) continue;
            c.c_plus_passes += 3;
            c.c_plus_elems += 3 * static_cast<int64_t>(qm) * qn;
            c.c_plus_flops += 2 * static_cast<int64_t>(qm) * qn;
        }
    }
}

void add_counters(strassen_counter_values& acc, const strassen_counter_values& d) {
    int64_t* a = &acc.pack_a_calls;
    const int64_t* b = &d.pack_a_calls;
    for (int i = 0; i < 19; ++i) a[i] += b[i];
}

// ------------------------------------------------------------------- model --
void validate_blocking(const strassen_blocking& p) {
    if (p.mc <= 0 || p.nc <= 0 || p.kc <= 0 || p.mr <= 0 || p.nr <= 0)
        throw std::invalid_argument("blocking: all parameters must be > 0");
    if (p.mc % p.mr != 0 || p.nc % p.nr != 0)
        throw std::invalid_argument("blocking: mc % mr and nc % nr must be 0");
    if (p.mr > 32 || p.nr > 32) throw std::invalid_argument("blocking: register tile too large");
}

static void validate_model(const strassen_model_params& p) {
    if (p.tau_a <= 0.0 || p.tau_b <= 0.0)
        throw std::invalid_argument("model: tau_a and tau_b must be > 0");
    if (p.lambda < 0.5 || p.lambda > 1.0)
        throw std::invalid_argument("model: lambda must be in [0.5, 1]");
}

double effective_gflops(long m, long n, long k, double seconds) {
    if (seconds <= 0.0) throw std::domain_error("effective_gflops: time must be > 0");
    return 2.0 * m * n * k / seconds * 1e-9;
}

namespace {
struct Coef {
    long a_mul, b_mul, c_mul, a_add, b_add, c_add;
};
Coef coefficients(strassen_variant v, int level) {
    if (level == 0 || v == STRASSEN_DGEMM) return {1, 1, 1, 0, 0, 0};
    if (level == 1) {
        if (v == STRASSEN_ABC) return {12, 12, 12, 0, 0, 0};
        if (v == STRASSEN_AB) return {12, 12, 7, 0, 0, 36};
        if (v == STRASSEN_NAIVE) return {7, 7, 7, 19, 19, 36};
    }
    if (level == 2) {  // the paper's figures (model.cpp:59-66)
        if (v == STRASSEN_ABC) return {194, 194, 154, 0, 0, 0};
        if (v == STRASSEN_AB) return {194, 194, 49, 0, 0, 462};
        if (v == STRASSEN_NAIVE) return {49, 49, 49, 293, 293, 462};
    }
    throw std::invalid_argument("model: unsupported variant configuration");
}
void op_counts(int level, long& mul, long& a, long& b, long& c) {
    switch (level) {
        case 0: mul = 1, a = 0, b = 0, c = 0; return;
        case 1: mul = 7, a = 5, b = 5, c = 12; return;
        case 2: mul = 49, a = 95, b = 95, c = 154; return;  // model.cpp:31
        default: throw std::invalid_argument("model: level must be 0, 1 or 2");
    }
}
}  // namespace

void model_predict(strassen_variant v, int level, long m, long n, long k,
                   const strassen_blocking& bp, const strassen_model_params& mp,
                   strassen_breakdown& out, double& egf) {
    if (m < 1 || n < 1 || k < 1) throw std::invalid_argument("model: dimensions must be >= 1");
    validate_model(mp);
    strassen_breakdown t{};
    // arithmetic (model.cpp:70-87)
    if (level == 0 || v == STRASSEN_DGEMM) {
        t.ta_mul = 2.0 * m * n * k * mp.tau_a;
    } else {
        long cm, ca, cb, cc;
        op_counts(level, cm, ca, cb, cc);
        const long s = 1L << level;
        const long qm = ceil_div(m, s), qn = ceil_div(n, s), qk = ceil_div(k, s);
        t.ta_mul = cm * 2.0 * qm * qn * qk * mp.tau_a;
        t.ta_a_add = ca * 2.0 * qm * qk * mp.tau_a;
        t.ta_b_add = cb * 2.0 * qk * qn * mp.tau_a;
        t.ta_c_add = cc * 2.0 * qm * qn * mp.tau_a;
    }
    // memory (model.cpp:89-111)
    validate_blocking(bp);
    const Coef cs = coefficients(v, level);
    const int lvl = (v == STRASSEN_DGEMM) ? 0 : level;
    const long s = 1L << lvl;
    const long qm = ceil_div(m, s), qn = ceil_div(n, s), qk = ceil_div(k, s);
    const double tb = mp.tau_b * mp.channel_factor;
    t.tm_a_mul = cs.a_mul * static_cast<double>(qm) * qk * ceil_div(qn, bp.nc) * tb;
    t.tm_b_mul = cs.b_mul * static_cast<double>(qn) * qk * tb;
    t.tm_c_mul = cs.c_mul * mp.lambda * 2.0 * qm * qn * ceil_div(qk, bp.kc) * tb;
    t.tm_a_add = cs.a_add * static_cast<double>(qm) * qk * tb;
    t.tm_b_add = cs.b_add * static_cast<double>(qn) * qk * tb;
    t.tm_c_add = cs.c_add * static_cast<double>(qm) * qn * tb;
    t.total = (t.ta_mul + t.ta_a_add + t.ta_b_add + t.ta_c_add) +
              (t.tm_a_mul + t.tm_b_mul + t.tm_c_mul + t.tm_a_add + t.tm_b_add + t.tm_c_add);
    out = t;
    egf = effective_gflops(m, n, k, t.total);
}


// ------------------------------------------------------- B200 dispatch model --
// The paper's purpose for its model is choosing the family member per shape
// (reference model.cpp).  This is the same T = T_a + T_m split
// re-fitted to B200 with the round-1 measurements (profiles/r01_notes.md,
// profiles/r01_sweep_*.csv):
//   T_a: executed mm_kernel flops / (37.05 TF/s * e_mm * wave efficiency), with
//        e_mm = 0.976 for single-term programs (DGEMM, Naive, C), 0.91 / 0.78 for
//        the fused two- / four-term sums (ABC, AB at level 1 / 2);
//   T_m: HBM bytes of the sum / stream traffic at 5.5 TB/s, and the fused
//        epilogue's reduce-add traffic at an effective 20 (single-term, deferred)
//        or 10 TB/s (fused sums) -- constants fitted by tools/model_fit.py;
//   + 20 us per dependent launch (drain of one kernel and ramp of the next,
//     fitted to the small sweep sizes) and the split-mode partials for outputs
//     under two waves.
namespace {
double waves_eff(double ctas, double sms) {
    const double w = std::ceil(ctas / sms);
    return ctas / (w * sms);
}
}  // namespace

// c_vec: C column-major with an even ldc and 16-byte aligned quadrant origins
// (engine.cpp run_strassen), which the TMA reduce-add epilogue needs; otherwise
// the fused epilogue is the register read-modify-write.
static double predict_core(strassen_variant v, int L, long m, long n, long k, int sms,
                           bool c_vec) {
    const double P = 37.05e12, BW = 5.5e12, launch = 12e-6;
    const long S = 1L << L;
    const double qm = static_cast<double>(ceil_div(m, S)), qn = static_cast<double>(ceil_div(n, S)),
                 qk = static_cast<double>(ceil_div(k, S));
    static const double tc[3][4] = {{1, 0, 0, 1}, {7, 5, 5, 12}, {49, 95, 95, 144}};
    static const double n_sums[3] = {0, 5, 45};  // multi-term operand sums per side
    const double mul = tc[L][0], cu = tc[L][3];
    // (C and Naive run 64-wide tiles where the last 128-wide tile column would be at most
    // half used, engine.cpp run_strassen: count the columns in halves there)
    const double rem_n = std::fmod(qn, 128.0);
    const bool half_edge = (v == STRASSEN_C || v == STRASSEN_NAIVE || (v == STRASSEN_AB && L == 2)) &&
                           rem_n > 0 && rem_n <= 64 &&
                           std::ceil(qn / 128.0) <= 15 && std::ceil(qk / 16.0) <= 128;
    const double tiles = std::ceil(qm / 128.0) *
                         (half_edge ? std::ceil(qn / 64.0) / 2.0 : std::ceil(qn / 128.0));
    // mm_kernel efficiency (executed flops / DMMA peak), fitted to the sweeps
    // (tools/model_fit.py, profiles/r02_sweep_*.csv): single-term 0.976; fused operand
    // sums 0.91 at level 1; at level 2 the 4-term sides are materialised (the default
    // fused-term setting, 2) and the rest fused: E_ABC2
    const bool fused_sums = v == STRASSEN_ABC || v == STRASSEN_AB;
    constexpr double E_ABC2 = 0.93;
    double e_mm = 0.976;
    if (fused_sums) e_mm = (L == 1) ? 0.91 : E_ABC2;
    const bool per_product_grid = (v == STRASSEN_AB || v == STRASSEN_NAIVE);
    // k-chunks and the fused / split decision as engine.cpp plan_fused makes them
    const double terms = fused_sums ? (L == 1 ? 1.71 : 2.94) : 1.0;
    const double ks_fit = choose_ksplit(static_cast<long>(tiles), static_cast<long>(mul),
                                        static_cast<long>(std::ceil(qk / 16.0)), sms, qm * qn,
                                        1.0 + 0.15 * (terms - 1.0), nullptr);
    const bool fused = tiles >= 2.0 * sms || (mul > 1 && ks_fit == 1 && tiles >= sms);
    const bool split = !fused;
    // fused epilogue with several products: one CTA per (tile, product), ticketed
    double ctas = (per_product_grid || split || mul > 1) ? tiles * mul : tiles;
    double ks = 1;
    if (per_product_grid || split) {
        ks = ks_fit;
        ctas *= ks;
    }
    // executed flops: whole 128 x 128 x 16 tile steps -- partial tiles at the quadrant
    // edges run padded (2304^3 at level 2: quadrants of 576 = 4.5 tiles, 23% more work;
    // profiles/r02_mid_scan_variants.log)
    const double flops_q = tiles * 128.0 * 128.0 * std::ceil(qk / 16.0) * 16.0;
    // per-CTA fixed cost (barrier init, pipeline fill, epilogue): ~4 us per wave
    double t = mul * 2.0 * flops_q / (P * e_mm * waves_eff(ctas, sms)) +
               4e-6 * std::ceil(ctas / sms);
    if (mul == 1 && fused && tiles < 4.0 * sms) {
        // classical launches of two to four waves of tiles: stream-K over all the tiles
        // where engine.cpp plan_fused's comparison says so; 2.22 us per k-step and the
        // pieces' fixup fitted to profiles/r02_streamk_wide_ab.log (2304^3 734 us,
        // 2816^3 1303 us back to back)
        const double kt = std::ceil(qk / 16.0), total = tiles * kt;
        const double len = std::ceil(total / std::max(1.0, std::min<double>(sms, std::floor(total / 8))));
        const double t_k = 2.1e-6, t_cta = 3e-6;
        const double t_uni = std::ceil(tiles / sms) * (kt * t_k + t_cta);
        const double t_sk = len * t_k + std::ceil(len / kt + 1.0) * t_cta + 15e-6;
        if (t_sk < 0.97 * t_uni) t = len * 2.22e-6 + 14e-6;
    }
    if (mul == 1 && fused && tiles >= 4.0 * sms) {
        // four waves and more: whole waves of tile owners plus a stream-K tail where
        // plan.hpp choose_tail finds one (engine.cpp plan_fused), scaled from its estimate
        const long tm = static_cast<long>(std::ceil(qm / 128.0)), tn = static_cast<long>(std::ceil(qn / 128.0));
        const long kt = static_cast<long>(std::ceil(qk / 16.0));
        const TailPlan T = choose_tail(tm, tn, kt, sms);
        if (T.cols > 0)
            t *= T.t / (std::ceil(tiles / sms) * (static_cast<double>(kt) * 2.1e-6 + 3e-6));
    }
    if (mul > 1 && split && tiles * mul < 4.0 * sms) {
        // stream-K pieces of the (product, tile, k-step) space, as engine.cpp plan_fused
        // decides them; the pieces run at ~0.8 of the mainloop rate at these sizes
        // (per-piece prologue / fixup, profiles/r02_small6.log)
        const double kt = std::ceil(qk / 16.0), total = tiles * mul * kt;
        const double len = std::ceil(total / std::max(1.0, std::min<double>(sms, std::floor(total / 8))));
        const double t_k = 2.1e-6 * (1.0 + 0.15 * (terms - 1.0)), t_cta = 3e-6;
        const double per = std::ceil(kt / ks);
        const double t_uni = std::ceil(tiles * mul * ks / sms) * (per * t_k + t_cta);
        const double t_sk = len * t_k + std::ceil(len / kt + 1.0) * t_cta + 6e-6;
        if (t_sk < 0.97 * t_uni)
            t = mul * 2.0 * flops_q / (P * e_mm * 0.8 * waves_eff(std::ceil(total / len), sms)) +
                std::ceil(len / kt + 1.0) * 4e-6;
    }
    if (mul == 1 && split) {  // stream-K pieces when they beat the k-chunk waves (engine.cpp)
        const double kt = std::ceil(qk / 16.0), total = tiles * kt;
        const double len = std::ceil(total / std::max(1.0, std::min<double>(sms, std::floor(total / 8))));
        const double per = std::ceil(kt / ks), t_k = 2.1e-6, t_cta = 3e-6;
        const double t_uni = std::ceil(tiles * ks / sms) * (per * t_k + t_cta) +
                             (ks > 1 ? 15e-6 : 0.0);
        const double t_sk = len * t_k + t_cta + 15e-6;
        // (the decision as engine.cpp makes it; the time it takes carries the pieces'
        // measured fixup, ~35 us: 1024^3 94 us back to back)
        if (t_sk < 0.97 * t_uni) t = t_sk + 20e-6;
    }
    double bytes = 0.0;
    int launches = 1;
    if (v == STRASSEN_NAIVE || v == STRASSEN_C) {  // gather-form sum passes, both sides:
        const double quads = S * S + n_sums[L];     // sources read once, sums written once
        bytes += 8.0 * quads * (qm * qk + qk * qn);
        launches += 2;
    } else if (fused_sums && L == 2) {  // the 25 four-term sides of each operand
        bytes += 8.0 * (S * S + 25.0) * (qm * qk + qk * qn);
        launches += 2;
    }
    double rmw_bytes = 0.0;
    if (mul == 1 && split) {  // classical: partials summed by the last piece's CTA, no
        // stream pass (engine.cpp plan_fused fixup / stream-K)
        bytes += 8.0 * (1.5 * ks * qm * qn + 2.0 * m * n);
    } else if (per_product_grid || split) {  // M_{p,s} written (mostly hidden under the
        // DMMAs), then read once by the stream pass with C read and written once
        bytes += 8.0 * (1.5 * ks * mul * qm * qn + 2.0 * m * n);
        launches += 1;
    } else {  // fused epilogue: C read + written at L2 per C update (TMA reduce-adds),
        // mostly hidden: persistent single-term launches collect them a unit later
        // short products of ABC / C run in groups of up to three products per unit whose
        // shared destinations take one update (engine.cpp pair_products): the level-1/2
        // tables' 12 / 144 updates become 7 / 90.  Credited where the updates bound the
        // call (<= 8 k-tiles: 16384^2 x 256 ABC L2 9.1 -> 6.7 ms); at 16 k-tiles they
        // are mostly hidden already (x 1024: 16.5 -> 16.1, profiles/r02_group14_*.log)
        const bool grouped = (v == STRASSEN_ABC || v == STRASSEN_C) && mul > 1 &&
                             std::ceil(qk / 16.0) <= 8;
        rmw_bytes = 16.0 * (grouped ? (L == 1 ? 7.0 : 90.0) : cu) * qm * qn;
    }
    // the deferred (persistent, separate-stage) epilogue: single-term programs, and
    // fused ones whose sides are at most 2 terms with short products (engine.cpp)
    const bool deferred = !fused_sums || (L == 2 && std::ceil(qk / 16.0) <= 8);
    t += bytes / BW + rmw_bytes / (!c_vec ? 4.6e12 : deferred ? 20e12 : 10e12) +
         launches * launch;
    return t;
}

// Level 3 (Naive / C, engine.cpp run_outer): the outer operand sums (four source
// quadrants read, five sums written per side), the products zeroed, seven level-2
// calls on the outer quadrants, and the outer stream pass (seven M_r read, C read
// and written), at the HBM rate of the level-2 passes.
static double predict_level3(strassen_variant v, long m, long n, long k, int sms) {
    const double BW = 5.5e12, launch = 20e-6;
    const long qm = ceil_div(m, 2), qn = ceil_div(n, 2), qk = ceil_div(k, 2);
    const double bytes = 8.0 * 9.0 * (static_cast<double>(qm) * qk + static_cast<double>(qk) * qn) +
                         8.0 * 7.0 * qm * qn +
                         8.0 * (7.0 * qm * qn + 2.0 * static_cast<double>(m) * n);
    return 7.0 * b200_predict_seconds(v, 2, qm, qn, qk, sms) + bytes / BW + 4 * launch;
}

double b200_predict_seconds(strassen_variant v, int level, long m, long n, long k, int sms) {
    if (level == 3 && (v == STRASSEN_NAIVE || v == STRASSEN_C)) {
        // peeling as run_device does at level 3 (fringe kernels for the three updates)
        const long me = peel_core(m, 8, 128, 16), ne = peel_core(n, 8, 128, 16), ke = k & ~7L;
        auto work3 = [&](long mm, long nn, long kk) {
            return ceil_div(ceil_div(mm, 8), 128) * ceil_div(ceil_div(nn, 8), 128) *
                   ceil_div(ceil_div(kk, 8), 16);
        };
        if ((me != m || ne != n || ke != k) && me >= 8 * 128 && ne >= 8 * 128 && ke >= 8 * 16 &&
            m - me <= 16 && n - ne <= 16 &&
            peel_pays(work3(m, n, k), work3(me, ne, ke), 343, sms, fringe_bytes(m, n, k, me, ne, ke))) {
            const double BWF = 4.5e12, launch = 12e-6;
            double t = predict_level3(v, me, ne, ke, sms);
            if (ke < k) t += 16.0 * me * ne / BWF + launch;
            if (me < m) t += 8.0 * static_cast<double>(k) * n / BWF + 2 * launch;
            if (ne < n) t += 8.0 * static_cast<double>(me) * k / BWF + 2 * launch;
            return t;
        }
        return predict_level3(v, m, n, k, sms);
    }
    const int L = (v == STRASSEN_DGEMM) ? 0 : level;
    const long S = 1L << L;
    // (the fringe kernels' width, fringe.cu kThinMax)
    const long me = peel_core(m, S, 128, 16), ne = peel_core(n, S, 128, 16), ke = k & ~(S - 1);
    // dynamic peeling as engine.cpp run_device applies it: the even core, then
    // three classical fringe updates
    auto work = [&](long mm, long nn, long kk) {
        return ceil_div(ceil_div(mm, S), 128) * ceil_div(ceil_div(nn, S), 128) *
               ceil_div(ceil_div(kk, S), 16);
    };
    // column-major C with ldc = m: an odd m, or odd quadrant rows, rule out the
    // 16-byte epilogue
    auto vec = [&](long rows) { return m % 2 == 0 && (L == 0 || ceil_div(rows, S) % 2 == 0); };
    if ((me != m || ne != n || ke != k) && me >= S * 128 && ne >= S * 128 && ke >= S * 16 &&
        m - me <= 16 && n - ne <= 16 &&
        peel_pays(work(m, n, k), work(me, ne, ke), L == 0 ? 1 : L == 1 ? 7 : 49, sms,
                  fringe_bytes(m, n, k, me, ne, ke))) {
        double t = predict_core(v, L, me, ne, ke, sms, vec(me));
        // the fringe updates are streaming kernels (fringe.cu): the long operand or C
        // once through HBM (4.5 TB/s measured at 4097^3 / 8193^3) plus their launches
        const double BWF = 4.5e12, launch = 12e-6;
        if (ke < k) t += 16.0 * me * ne / BWF + launch;
        if (me < m) t += 8.0 * static_cast<double>(k) * n / BWF + 2 * launch;
        if (ne < n) t += 8.0 * static_cast<double>(me) * k / BWF + 2 * launch;
        return t;
    }
    return predict_core(v, L, m, n, k, sms, vec(m));
}

void b200_select(long m, long n, long k, int sms, strassen_variant& v_out, int& l_out,
                 double& t_out, int max_level) {
    const struct {
        strassen_variant v;
        int l;
    } cand[] = {{STRASSEN_DGEMM, 0}, {STRASSEN_ABC, 1}, {STRASSEN_AB, 1}, {STRASSEN_NAIVE, 1},
                {STRASSEN_C, 1},     {STRASSEN_ABC, 2}, {STRASSEN_AB, 2}, {STRASSEN_NAIVE, 2},
                {STRASSEN_C, 2},     {STRASSEN_NAIVE, 3}, {STRASSEN_C, 3}};
    t_out = 1e300;
    for (const auto& c : cand) {
        if (c.l > max_level) continue;
        if (c.l > 0 && (m < (1L << c.l) || n < (1L << c.l) || k < (1L << c.l))) continue;
        const double t = b200_predict_seconds(c.v, c.l, m, n, k, sms);
        if (t < t_out) {
            t_out = t;
            v_out = c.v;
            l_out = c.l;
        }
    }
}

}  // namespace sb200
