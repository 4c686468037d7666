// Operation counters (reference: proj/include/qpack/counters.hpp:10-33).
//   mul_add          word multiply/accumulates in the main loops
//   divisions        divisions by p (one per REDQ, premultiplied or not)
//   table_accesses   lookup-table reads
//   reduction_calls  REDQ invocations
// Divisions by powers of q are shifts and are never counted.
#pragma once

#include <cstdint>

namespace qpack {

struct CostReport {
    std::uint64_t mul_add = 0;
    std::uint64_t divisions = 0;
    std::uint64_t table_accesses = 0;
    std::uint64_t reduction_calls = 0;

    CostReport& operator+=(const CostReport& other) {
        mul_add += other.mul_add;
        divisions += other.divisions;
        table_accesses += other.table_accesses;
        reduction_calls += other.reduction_calls;
        return *this;
    }
};

}  // namespace qpack
