// Per-rank amplitude-memory accounting — declaration-compatible with the
// reference proj/include/qsim/memtrack.hpp:8-26 (definitions in
// cpp/src/memtrack.cpp are independent).
//
// On the B200 build a "rank" is one GPU driven by one host thread (or one
// process under torchrun).  Device allocations made through the C-ABI
// (state shards, swap chunk buffers) are reported here by the calling thread,
// which is how the BBOP memory bound (2^l + B*2^b)*16 B (SPEC.md:343, :397,
// :573) is evidenced for HBM.
#pragma once

#include <cstddef>
#include <cstdint>

namespace qsim::memtrack {

// Working-set phases: the execution phase and the gather/scatter staging.
enum class Phase : int { execute = 0, gather = 1 };

// Global switch.  enable() sizes the table for `ranks` ranks and clears it.
void enable(int ranks);
void disable();
bool enabled();

// The calling thread's rank / phase (thread-local).
void register_thread(int rank);
void unregister_thread();
void set_phase(Phase phase);

// Record an allocation / release of amplitude storage by the calling thread.
void on_alloc(std::size_t bytes);
void on_free(std::size_t bytes);

// High-water mark of a rank in a phase; 0 for an unknown rank.
std::size_t peak_bytes(int rank, Phase phase);
// Zero every counter, keeping the rank table size.
void reset();

} // namespace qsim::memtrack
