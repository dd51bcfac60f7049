// Internal (non-ABI) structures shared by the libqsv translation units.
#pragma once

#include "qsv.h"

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <map>
#include <string>
#include <vector>

namespace qsv {

// One op compiled against the tile layout of its pass.  A pass is uploaded as
// one "blob" = [TileOp x nops][member-offset tables][matrices / diagonal
// tables]; each CTA copies the blob to shared memory once and every later read
// is a warp-broadcast LDS.
struct TileOp {
    int32_t kind;       // QSV_OP_*
    int32_t k;          // DENSE/XPERM: number of targets; DIAG: number of qubits
    int32_t nfix;       // number of sorted positions in fixpos[]
    uint32_t tctrl;     // tile-local control bits (must be 1)
    uint64_t xctrl;     // full-index control bits outside the tile (CTA-uniform test)
    uint32_t mat_byte;  // byte offset (in the blob) of the matrix / diagonal table
    uint32_t off_byte;  // DENSE: byte offset of the 2^k member-offset table (uint32)
    uint32_t tmask;     // DIAG: tile positions of the in-tile qubits (table bits 0..nin-1)
    int32_t nin;        // DIAG: number of in-tile qubits
    int8_t tpos[QSV_MAX_DIAG_K];  // DENSE/XPERM: tile-local position of target i
    int8_t xbit[QSV_MAX_DIAG_K];  // DIAG: full-index bit of out-of-tile qubit j (table bit nin+j)
    int8_t fixpos[24];            // ascending tile positions fixed during group enumeration
    uint32_t fmask;               // OR of 1 << fixpos[i]
    uint32_t ptab_byte;           // DIAG: byte offset of pext tables (uint8 [32] low, [64] high)
    uint32_t prim_byte;           // RBLOCK: DevPrim list; PHASEPROD: ExtFactor list
    int32_t nprim;
    uint32_t rot_tab;             // RBLOCK: 4-bit member rotation per lane & 7 (bank spreading)
    uint32_t pad2[3];
};

// RBLOCK primitive as stored in the blob.
struct DevPrim {
    uint8_t kind;       // QSV_PRIM_U1 / U2 / CX / DIAG16
    uint8_t a, b;       // block-local qubit indices (0..3)
    uint8_t pad;
    uint32_t data_byte; // blob offset of the matrix / table; U1 stores 2 variants
                        // (U, XUX), U2 stores 4 (conjugated by X on a, b), one per
                        // member rotation of the lane
};

// PHASEPROD factor on a qubit outside the tile (CTA-uniform).
struct ExtFactor {
    double re, im;
    int32_t bit;        // full-index bit
    int32_t pad[3];
};
static_assert(sizeof(TileOp) % 16 == 0, "TileOp must keep 16-B alignment in the blob");

// Largest per-pass blob (bytes of shared memory on top of the tile buffers).
constexpr uint32_t kMaxBlobBytes = 40 * 1024;

// Tile geometry of one pass: tile = [0, L) U {high[0..nhigh)} in local index bits.
struct PassGeom {
    int32_t K;        // tile qubits
    int32_t L;        // contiguous low run
    int32_t nhigh;
    int32_t high[QSV_MAX_HIGH];
    int32_t kmax;     // largest dense arity in the pass (selects the kernel variant)
};

struct Step {
    qsv_step_desc desc;
    PassGeom geom{};
    int nops = 0;
    uint64_t blob_off = 0;   // byte offset of this pass's blob in Program::d_blobs
    uint32_t blob_bytes = 0;
    double hbm_bytes = 0, flops = 0, nvl_bytes = 0;
};

} // namespace qsv

struct qsv_ctx {
    int device = 0;
    int rank = 0;
    int nranks = 1;
    int sm_count = 0;
    cudaStream_t stream = nullptr;      // compute stream (all public work is ordered here)
    cudaStream_t comm_stream = nullptr; // NCCL transfers of a swap
    cudaStream_t copy_stream = nullptr; // staging copy-back of a swap
    cudaEvent_t ev_a = nullptr, ev_b = nullptr;
    ncclComm_t comm = nullptr;
    // reduction scratch
    double* d_partials = nullptr;
    double* h_result = nullptr;   // pinned, 4 doubles
    size_t partials_cap = 0;
    // swap staging (nbuf chunks)
    void* d_stage = nullptr;
    size_t stage_bytes = 0;
    // host->device scratch for diff checks
    double* d_scratch = nullptr;
    size_t scratch_bytes = 0;
};

struct qsv_state {
    qsv_ctx* ctx = nullptr;
    int n_local = 0;
    uint64_t size = 0;     // 2^n_local amplitudes
    double2* amps = nullptr;
};

struct qsv_program {
    qsv_ctx* ctx = nullptr;
    int n_total = 0, n_local = 0;
    std::vector<qsv::Step> steps;
    unsigned char* d_blobs = nullptr;
    size_t blob_total = 0;
    bool has_collective = false;
    // one captured graph per state buffer it was run on
    std::map<const void*, cudaGraphExec_t> graphs;
};

namespace qsv {
void set_error(const std::string& msg);
// Launches the pass kernel variant for `geom` on `st` (compute stream).
cudaError_t launch_pass(const qsv_state* st, const Step& step, const unsigned char* d_blob,
                        uint64_t rank_base, cudaStream_t stream);
// Runs one chunked qubit swap (BBOP) of `st` with its peer; see qsv_swap.
int run_swap(qsv_state* st, int g, int v, int chunk_log2, int nbuf);
} // namespace qsv
