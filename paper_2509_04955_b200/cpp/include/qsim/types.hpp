// qsim core scalar types — declaration-compatible with the reference header
// proj/include/qsim/types.hpp:9-19 so reference callers compile unchanged.
//
// Layout contract: an amplitude is two IEEE fp64
// values (re, im) = 16 bytes, and qubit k is bit k of the amplitude index
// (little-endian).  std::complex<double> is layout-compatible with CUDA's
// double2, which is what lets a host Amp* be handed straight to the C-ABI
// in include/qsv.h.
#pragma once

#include <complex>
#include <cstdint>

namespace qsim {

using Amp = std::complex<double>;   // ref types.hpp:9
using Index = std::uint64_t;        // ref types.hpp:10

static_assert(sizeof(Amp) == 16, "amplitude must be 16 bytes (SPEC.md:32)");

// 2^k as an index value (ref types.hpp:12).
constexpr Index index_bit(int k) { return Index{1} << k; }

// Spread j so that bit position k becomes a zero and the bits of j at and
// above k move one place up (ref types.hpp:14-19).  With j enumerating
// 0..2^{n-1}-1 this yields the lower member of every amplitude pair of a
// gate on qubit k (Alg. 3 "group" traversal).
constexpr Index insert_zero_bit(Index j, int k) {
    const Index below = index_bit(k) - 1;
    return (j & below) | ((j & ~below) << 1);
}

} // namespace qsim
