// Reference-parity instrumentation counters and analytical model (host only).
#pragma once
#include "strassen.h"

namespace sb200 {

// Adds to `c` the counter values the reference would record for one
// strassen_gemm call with blocking `bp` (counters.hpp:8-49 semantics).
void count_call(strassen_variant variant, int level, long m, long n, long k,
                const strassen_blocking& bp, strassen_counter_values& c);
void add_counters(strassen_counter_values& acc, const strassen_counter_values& d);

// Throws std::invalid_argument like BlockingParams::validate (kernel.hpp:20-27).
void validate_blocking(const strassen_blocking& p);

// model.cpp:113-117; throws std::domain_error when seconds <= 0.
double effective_gflops(long m, long n, long k, double seconds);

// model.cpp:119-134.
void model_predict(strassen_variant v, int level, long m, long n, long k,
                   const strassen_blocking& bp, const strassen_model_params& mp,
                   strassen_breakdown& out, double& egf);

// B200 cost model (strassen_select): predicted seconds of
// one strassen_gemm call, and the fastest (variant, level) for a shape.
double b200_predict_seconds(strassen_variant v, int level, long m, long n, long k, int sms);
// level 3 (Naive / C) is predicted for v in {NAIVE, C}; b200_select considers it only
// when max_level >= 3 (a ctx that admits it, strassen_ctx_select)
void b200_select(long m, long n, long k, int sms, strassen_variant& v_out, int& l_out,
                 double& t_out, int max_level = 2);

}  // namespace sb200
