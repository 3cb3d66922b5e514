// Strassen operand tables (host side, integer).
//
// Restates the reference's symbolic program (table.hpp:8-45, table.cpp:14-113):
// a one-level table of 7 products and Kronecker-style composition for higher
// levels.  Quadrant index = row * 2^L + col.  Level 2 is composed, never
// hand-entered, and is what the GPU product programs are built
// from (plan.cpp).
#pragma once
#include <stdexcept>
#include <utility>
#include <vector>

namespace sb200 {

using Terms = std::vector<std::pair<int, int>>;  // (quadrant, coefficient)

struct Product {
    Terms a, b, c;  // operand sums and C destinations
};

struct Program {
    int level = 0;
    std::vector<Product> products;  // 7^level
};

struct OpCounts {
    long mults = 0, a_adds = 0, b_adds = 0, c_updates = 0;
};

Program identity_program();
Program one_level_program();
// outer (x) inner; duplicates merged by coefficient addition, zeros dropped,
// coefficients must stay in {-1, 0, 1} (table.cpp:39-93).
Program compose(const Program& outer, const Program& inner);
// Level 1 or 2; throws std::invalid_argument otherwise (table.cpp:95-102).
const Program& program_for_level(int level);
// Level 3 = compose(level 1, level 2): 343 products (B200 extension; the
// reference composes it only in acceptance.cpp:86-88).  Used for the analytic
// counters of level-3 calls.
const Program& program_level3();
OpCounts count_ops(const Program& p);

}  // namespace sb200
