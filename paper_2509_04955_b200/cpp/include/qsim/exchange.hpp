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

#include <vector>

namespace qsim {

struct DistributedReport {
    int ranks = 1;
    std::size_t swaps = 0;
    double seconds = 0.0;             // wall time of the simulation (all ranks)
    std::vector<std::size_t> peak_bytes;  // per-rank device bytes (state + staging)
};

// Simulates `c` from |0...0> over plan.ranks() GPUs (devices[r] for rank r,
// default 0..ranks-1) and gathers the state to rank 0's host StateVector.
StateVector run_distributed(const Circuit& c, const PartitionPlan& plan, const std::vector<int>& devices = {},
                            DistributedReport* report = nullptr, const PlanOptions& opt = PlanOptions{});

} // namespace qsim
