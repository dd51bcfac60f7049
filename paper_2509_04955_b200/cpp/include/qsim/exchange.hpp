// Distributed execution: run_distributed.
// Ranks are GPUs driven by one host thread each (the SPEC's thread-per-rank
// model; memtrack's thread-local rank, ref memtrack.cpp:20-21).
// Global qubits are moved by chunked, double-buffered NVLink qubit swaps
// (BBOP, swap.cu) inserted by the planner; the result is gathered to the host.
#pragma once

#include "qsim/circuit.hpp"
#include "qsim/partition.hpp"
#include "qsim/planner.hpp"
#include "qsim/statevector.hpp"

#include <string>
#include <vector>

namespace qsim {

struct DistributedReport {
    int ranks = 1;
    std::size_t swaps = 0;
    double seconds = 0.0;             // wall time of the simulation (all ranks)
    // per-rank high-water mark of the library's device allocations (state shard, swap
    // staging, program blobs, scratch), instrumented through qsv_ctx_mem
    std::vector<std::size_t> peak_bytes;
    std::vector<std::string> files;   // run_distributed_to_files: one shard file per rank
};

// Largest state (bytes) run_distributed gathers to one host: QSV_GATHER_CAP_GIB
// (default 64 GiB).  Larger states are refused there; run_distributed_to_files writes one
// file per rank instead.
std::size_t gather_cap_bytes();

// Same simulation as run_distributed, but each rank writes its shard (global indices
// [r 2^l, (r+1) 2^l), interleaved little-endian fp64 re/im) to <dir>/shard_r<r>_of_<R>.bin
// and rank 0 writes <dir>/manifest.json; nothing is gathered.
void run_distributed_to_files(const Circuit& c, const PartitionPlan& plan, const std::string& dir,
                              const std::vector<int>& devices = {}, DistributedReport* report = nullptr,
                              const PlanOptions& opt = PlanOptions{});

// Simulates `c` from |0...0> over plan.ranks() GPUs (devices[r] for rank r,
// default 0..ranks-1) and gathers the state to rank 0's host StateVector.
StateVector run_distributed(const Circuit& c, const PartitionPlan& plan, const std::vector<int>& devices = {},
                            DistributedReport* report = nullptr, const PlanOptions& opt = PlanOptions{});

} // namespace qsim
