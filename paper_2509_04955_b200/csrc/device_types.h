// Device-visible data structures of a compiled pass, shared by the nvcc-built
// interpreter kernel (pass_kernel.cu) and the NVRTC-specialised pass kernels
// (jit.cu).  Must compile both as host C++ and under NVRTC (no host headers).
#pragma once

#if defined(__CUDACC_RTC__)
typedef unsigned char uint8_t;
typedef signed char int8_t;
typedef unsigned short uint16_t;
typedef int int32_t;
typedef unsigned int uint32_t;
typedef long long int64_t;
typedef unsigned long long uint64_t;
#else
#include <cstdint>
#endif

#if !defined(__CUDACC__) && !defined(__CUDACC_RTC__) && !defined(__align__)
#define __align__(n) alignas(n)
#endif

#ifndef QSV_H
// values mirror include/qsv.h (static_assert-checked in qsv_internal.h)
#define QSV_MAX_DENSE_K 5
#define QSV_MAX_DIAG_K 8
#define QSV_MAX_HIGH 8
#define QSV_MAX_TILE_K 12
#define QSV_OP_DENSE 0
#define QSV_OP_DIAG 1
#define QSV_OP_XPERM 2
#define QSV_OP_RBLOCK 3
#define QSV_OP_PHASEPROD 4
#define QSV_OP_PARPHASE 5
#define QSV_PRIM_U1 0
#define QSV_PRIM_U2 1
#define QSV_PRIM_CX 2
#define QSV_PRIM_DIAG16 3
#define QSV_PRIM_FACTOR 4
#define QSV_PRIM_U1R 5
#define QSV_PRIM_U1I 6
#endif

// Internal (device-only) op kind: the pass relabel appended after a pass's ops
// (qsv_step_desc::relabel); never appears in a qsv_op_desc.
#define QSV_OP_RELABEL 16
// Internal op kind: a 4-qubit register block whose primitive list is heavy enough is
// compiled on the host into its dense 16x16 unitary and applied with DMMA (FP64
// tensor-core mma.m8n8k4) instead of DFMA primitives.
#define QSV_OP_DMMA16 17

namespace qsv {

// One op compiled against the tile layout of its pass.  A pass is uploaded as
// one "blob" = [TileOp x nops][member-offset tables][matrices / diagonal
// tables]; each CTA copies the blob to shared memory once and every later read
// is a warp-broadcast LDS.
struct TileOp {
    int32_t kind;       // QSV_OP_*
    int32_t k;          // DENSE/XPERM: number of targets; DIAG: number of qubits; RBLOCK: slots
    int32_t nfix;       // number of sorted positions in fixpos[]
    uint32_t tctrl;     // tile-local control bits (must be 1)
    uint64_t xctrl;     // full-index control bits outside the tile (CTA-uniform test)
    uint32_t mat_byte;  // byte offset (in the blob) of the matrix / diagonal table
    uint32_t off_byte;  // DENSE: byte offset of the 2^k member-offset table (uint32)
    uint32_t tmask;     // DIAG: tile positions of the in-tile qubits (table bits 0..nin-1)
    int32_t nin;        // DIAG: number of in-tile qubits
    int8_t tpos[QSV_MAX_DIAG_K];  // DENSE/XPERM/RBLOCK: tile-local position of target/slot i
    int8_t xbit[QSV_MAX_DIAG_K];  // DIAG: full-index bit of out-of-tile qubit j (table bit nin+j)
    int8_t fixpos[24];            // ascending tile positions fixed during group enumeration
    uint32_t fmask;               // OR of 1 << fixpos[i]
    uint32_t ptab_byte;           // DIAG: byte offset of pext tables (uint8 [32] low, [64] high)
    uint32_t prim_byte;           // RBLOCK: DevPrim list; PHASEPROD: ExtFactor list
    int32_t nprim;
    uint32_t rot_tab;             // RBLOCK: 4-bit member rotation per lane & 7 (bank spreading)
    uint32_t pad2;
    uint64_t xmask;               // PARPHASE: out-of-tile qubits of the parity mask (full index)
};
static_assert(sizeof(TileOp) % 16 == 0, "TileOp must keep 16-B alignment in the blob");

// RBLOCK primitive as stored in the blob.
struct DevPrim {
    uint8_t kind;       // QSV_PRIM_U1 / U1R / U1I / U2 / CX / DIAG16
    uint8_t a, b;       // block-local qubit indices (0..3)
    uint8_t pad;
    uint32_t data_byte; // blob offset of the matrix / table; 2x2 kinds store 2 variants
                        // (U, XUX), U2 stores 4 (conjugated by X on a, b), one per
                        // member rotation of the lane
};

// PHASEPROD factor on a qubit outside the tile (CTA-uniform).
struct ExtFactor {
    double re, im;
    int32_t bit;        // full-index bit
    int32_t pad[3];
};

// Tile geometry of a pass as passed to the kernels.
struct GeomArg {
    int32_t L, nhigh;
    int32_t high[QSV_MAX_HIGH];
    uint64_t tile0;  // first tile of the launch (region launches overlapped with a swap)
    // region launch: tiles whose bits reg[0..nreg) (ascending, outside the tile) equal
    // rval; the tile index then enumerates the remaining bits only
    int32_t nreg;
    int32_t reg[3];
    uint64_t rval;
    // Fused qubit swap (BBOP over NVLink P2P, swap.cu / pass_pipeline): with `peer` set,
    // the pass runs on the layout AFTER swapping the global qubit of bit value `sgbit`
    // into local bit `sv`: the half of each tile (sv_tile = 1: sv is a high tile bit) or
    // the tiles (sv_tile = 0) whose bit sv differs from sgbit are read from the peer's
    // shard at index ^ (1 << sv); results are stored locally.  Before storing into a slot
    // the peer still has to read, a CTA waits for its twin (same blockIdx, same
    // iteration on the peer) to flag that its loads landed.
    const double2* peer;
    unsigned long long* flag_mine;  // written by the peer's twins
    unsigned long long* flag_peer;  // this rank's twins write here
    uint64_t epoch;                 // flag value of iteration i: (epoch << 32) | (i + 1)
    int32_t sv, sv_tile, sv_tidx;   // sv_tidx (sv_tile = 0): tile-index bit of sv
    uint32_t sgbit;
    // push mode (QSV_FUSE_SWAP=2): the swap is fused into the pass BEFORE it instead: loads are
    // local (pre-swap layout) and the runs whose bit sv differs from sgbit are stored into the
    // peer's shard at index ^ (1 << sv) (posted NVLink writes), after the twin flagged that it
    // has loaded those slots
    int32_t spush;
    // debug (QSV_DEBUG_POISON=1): every tile buffer run is filled with NaN before its
    // TMA load is issued, so an op that reads SMEM the load has not yet written (a broken
    // mbarrier / bulk-copy ordering) turns the result into NaN instead of a stale value
    int32_t poison;
    // Tensor-map tile copies (JIT kernels): with tm_rank > 0 the tile moves as 2^tm_nx
    // cp.async.bulk.tensor copies of a rank-tm_rank box instead of one bulk copy per
    // contiguous run.  Dim d covers amplitude-index bits [tm_s[d], tm_s[d + 1]) (the last
    // up to n_local); its box is the tile run starting at tm_s[d].  The tile bits above
    // the last boxed run (tm_x[0..tm_nx)) are iterated, one copy per value.
    int32_t tm_rank;
    int32_t tm_s[5];
    int32_t tm_nx;
    int32_t tm_x[QSV_MAX_HIGH];
    uint32_t tm_box_amps;
    int32_t pad_;
};

// The 128-byte CUDA tensor map (CUtensorMap), passed to the specialised kernels as a
// __grid_constant__ parameter (opaque here).
struct __align__(64) TmaDesc {
    unsigned long long v[16];
};

// Largest per-pass blob (bytes of shared memory on top of the tile buffers).
constexpr uint32_t kMaxBlobBytes = 40 * 1024;
// Tile buffers per CTA (TMA double buffering).
constexpr int kNumBuf = 2;

} // namespace qsv
