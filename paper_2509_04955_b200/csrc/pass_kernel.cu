// The fused multi-block pass kernel (sm_100a).
//
// One launch = one HBM round trip over a rank's shard.  This is the B200
// realisation of three reference ideas at once:
//   * apply_multi / Alg. 1-4 (Eq. 3/4 :124-169):
//     a dense 2^k x 2^k block applied to every 2^k-amplitude group;
//   * SMGP: many blocks applied per pass — here
//     every block of the pass is applied to an SMEM-resident tile in program
//     order, which makes the result bitwise equal to sequential application
//     (stronger than the SPEC's Latin-rotation schedule);
//   * DAGC outputs: the blocks are the fused gates.
//
// Tile = 2^K amplitudes: the contiguous low index run [0, L) (512-B+ DRAM
// runs for L >= 5) plus the `nhigh` high qubits the pass's dense blocks
// target.  The kernel is persistent (grid = resident CTAs) and software
// pipelined through NBUF tile buffers:
//
//   thread 0:  cp.async.bulk global->smem of the 2^nhigh runs of tile i+NBUF-1
//              (TMA bulk engine, completion on an mbarrier with expect_tx),
//              cp.async.bulk smem->global of tile i after its compute;
//   all:       wait on the mbarrier of tile i, apply the pass's ops, barrier.
//
// Bytes in flight therefore do not depend on how many registers the compute
// needs.  The pass's ops, member-offset tables and matrices ("blob") are copied
// to SMEM once per CTA; every op read afterwards is a warp-broadcast LDS.
//
// Ops:  DENSE (k <= 5 targets in the tile, controls anywhere), DIAG (2^k-entry
// diagonal on any qubits, incl. out-of-tile and rank bits: RZ/CP/CZ/S/T chains
// never force a qubit into the tile), XPERM (X / CX / Toffoli as an SMEM swap).
// Tile-bit controls restrict the group enumeration (Alg. 4's half-work,
// PAPER:238-257); out-of-tile controls are a CTA-uniform test of the tile base.
#include <string>
#include "qsv_internal.h"
#include "pass_device.cuh"

#include <algorithm>
#include <cstdlib>

namespace qsv {

namespace {

// Resident CTAs per SM the register allocation must allow.
template <int KMAX, int NT>
constexpr int min_ctas() {
    return NT < 128 ? 1 : (KMAX <= 3 ? 5 : (KMAX == 4 ? 3 : 1));
}

// Interpreter: walks the pass's TileOp records in SMEM.
template <int K, int KMAX, int NT>
__global__ void __launch_bounds__(NT, min_ctas<KMAX, NT>())
pass_kernel(double2* __restrict__ psi, const unsigned char* __restrict__ gblob, uint32_t blob_bytes,
            int nops, const __grid_constant__ GeomArg geom, uint64_t rank_base, uint64_t ntiles) {
    pass_pipeline<K, NT>(psi, gblob, blob_bytes, geom, rank_base, ntiles,
                         [&](double2* tile, const unsigned char* blob, uint64_t full_base) {
        const TileOp* ops = reinterpret_cast<const TileOp*>(blob);
        for (int o = 0; o < nops; ++o) {
            const TileOp& op = ops[o];
            if ((full_base & op.xctrl) != op.xctrl)
                continue;  // CTA-uniform: an out-of-tile control is 0 for this tile
            __syncthreads();
            if (op.kind == QSV_OP_DENSE) {
                const int kk = op.k;
                if (kk == 1) dense_op<1, K, NT>(tile, op, blob);
                if constexpr (KMAX >= 2 && K >= 2) { if (kk == 2) dense_op<2, K, NT>(tile, op, blob); }
                if constexpr (KMAX >= 3 && K >= 3) { if (kk == 3) dense_op<3, K, NT>(tile, op, blob); }
                if constexpr (KMAX >= 4 && K >= 4) { if (kk == 4) dense_op<4, K, NT>(tile, op, blob); }
                if constexpr (KMAX >= 5 && K >= 5) { if (kk == 5) dense5_op<K, NT>(tile, op, blob); }
            } else if (op.kind == QSV_OP_RBLOCK) {
                if constexpr (K >= 3) {
                    if (op.k == 3) rblock_op<K, NT, 3>(tile, op, blob);
                }
                if constexpr (K >= 4 && KMAX >= 4) {
                    if (op.k == 4) rblock_op<K, NT, 4>(tile, op, blob);
                }
            } else if (op.kind == QSV_OP_DMMA16) {
                if constexpr (K >= 4)
                    dmma16_op<K, NT>(tile, op, blob);
            } else if (op.kind == QSV_OP_PARPHASE) {
                parphase_op<K, NT>(tile, op, blob, full_base);
            } else if (op.kind == QSV_OP_PHASEPROD) {
                phaseprod_op<K, NT>(tile, op, blob, full_base);
            } else if (op.kind == QSV_OP_RELABEL) {
                relabel_op<K, NT>(tile, op, blob);
            } else if (op.kind == QSV_OP_DIAG) {
                diag_op<K, NT>(tile, op, blob, full_base);
            } else {
                xperm_op<K, NT>(tile, op);
            }
        }
    });
}

template <int K>
constexpr int threads_for() {
    return K >= 8 ? 128 : (K >= 6 ? 64 : 32);
}

template <int K, int KMAX>
cudaError_t launch_variant(const qsv_state* st, const Step& step, const unsigned char* d_blob,
                           uint64_t rank_base, cudaStream_t stream, const LaunchRange& rg) {
    constexpr int NT = threads_for<K>();
    constexpr size_t tile_smem = sizeof(double2) * kNumBuf * (size_t{1} << K);
    const size_t smem = tile_smem + step.blob_bytes;
    auto kern = pass_kernel<K, KMAX, NT>;
    static int configured_smem = 0;
    static int sm_count = 0;
    if (configured_smem < static_cast<int>(tile_smem + kMaxBlobBytes)) {
        const int want = static_cast<int>(tile_smem + kMaxBlobBytes);
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, want);
        if (e != cudaSuccess)
            return e;
        configured_smem = want;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev);
    }
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem);
    if (e != cudaSuccess)
        return e;
    if (per_sm < 1)
        per_sm = 1;
    GeomArg ga{};
    ga.L = step.geom.L;
    ga.nhigh = step.geom.nhigh;
    for (int i = 0; i < step.geom.nhigh; ++i)
        ga.high[i] = step.geom.high[i];
    const uint64_t all_tiles = st->size >> K;
    {
        static const int poison = [] {
            const char* e = std::getenv("QSV_DEBUG_POISON");
            return e && e[0] == '1' ? 1 : 0;
        }();
        ga.poison = poison;
    }
    if (rg.fuse) {
        ga.peer = rg.fuse->peer;
        ga.flag_mine = rg.fuse->flag_mine;
        ga.flag_peer = rg.fuse->flag_peer;
        ga.epoch = rg.fuse->epoch;
        ga.sv = rg.fuse->sv;
        ga.sv_tile = rg.fuse->sv_tile;
        ga.sv_tidx = rg.fuse->sv_tidx;
        ga.sgbit = rg.fuse->sgbit;
        ga.spush = rg.fuse->push;
    }
    const uint64_t region_tiles = apply_region(ga, rg, all_tiles);
    ga.tile0 = std::min(rg.tile0, region_tiles);
    const uint64_t tiles = std::min(rg.count, region_tiles - ga.tile0);
    if (tiles == 0)
        return cudaSuccess;
    const int sms = rg.sms > 0 ? std::min(rg.sms, sm_count) : sm_count;
    uint64_t grid = std::min<uint64_t>(tiles, static_cast<uint64_t>(per_sm) * sms);
    if (const char* g = std::getenv("QSV_DEBUG_GRID"))  // debug: fewer persistent CTAs, other tile order
        grid = std::max<uint64_t>(1, std::min<uint64_t>(grid, std::strtoull(g, nullptr, 10)));
    if (rg.fuse)  // one flag per CTA (kFlagBytes)
        grid = std::min<uint64_t>(grid, kFlagBytes / sizeof(unsigned long long));
    kern<<<static_cast<unsigned>(grid), NT, smem, stream>>>(st->amps, d_blob, step.blob_bytes,
                                                           step.nops, ga, rank_base, tiles);
    return cudaGetLastError();
}

template <int K>
cudaError_t launch_k(const qsv_state* st, const Step& step, const unsigned char* d_blob,
                     uint64_t rank_base, cudaStream_t stream, const LaunchRange& rg) {
    if constexpr (K >= 9) {
        switch (step.geom.kmax <= 1 ? 1 : step.geom.kmax) {
        case 1: return launch_variant<K, 1>(st, step, d_blob, rank_base, stream, rg);
        case 2: return launch_variant<K, 2>(st, step, d_blob, rank_base, stream, rg);
        case 3: return launch_variant<K, 3>(st, step, d_blob, rank_base, stream, rg);
        case 4: return launch_variant<K, 4>(st, step, d_blob, rank_base, stream, rg);
        default: return launch_variant<K, 5>(st, step, d_blob, rank_base, stream, rg);
        }
    } else {
        constexpr int KM = K < 5 ? K : 5;
        return launch_variant<K, KM>(st, step, d_blob, rank_base, stream, rg);
    }
}

} // namespace

uint64_t apply_region(GeomArg& ga, const LaunchRange& rg, uint64_t all_tiles) {
    ga.nreg = 0;
    ga.rval = rg.rval & rg.rmask;
    for (int b = 0; b < 64 && ga.nreg < 3; ++b)
        if ((rg.rmask >> b) & 1ull)
            ga.reg[ga.nreg++] = b;
    return all_tiles >> ga.nreg;
}

cudaError_t launch_pass(const qsv_state* st, const Step& step, const unsigned char* d_blob,
                        uint64_t rank_base, cudaStream_t stream, const LaunchRange& rg) {
    switch (step.geom.K) {
    case 1: return launch_k<1>(st, step, d_blob, rank_base, stream, rg);
    case 2: return launch_k<2>(st, step, d_blob, rank_base, stream, rg);
    case 3: return launch_k<3>(st, step, d_blob, rank_base, stream, rg);
    case 4: return launch_k<4>(st, step, d_blob, rank_base, stream, rg);
    case 5: return launch_k<5>(st, step, d_blob, rank_base, stream, rg);
    case 6: return launch_k<6>(st, step, d_blob, rank_base, stream, rg);
    case 7: return launch_k<7>(st, step, d_blob, rank_base, stream, rg);
    case 8: return launch_k<8>(st, step, d_blob, rank_base, stream, rg);
    case 9: return launch_k<9>(st, step, d_blob, rank_base, stream, rg);
    case 10: return launch_k<10>(st, step, d_blob, rank_base, stream, rg);
    case 11: return launch_k<11>(st, step, d_blob, rank_base, stream, rg);
    default:
        set_error("pass: tile_k " + std::to_string(step.geom.K) +
                  " has no interpreter kernel (only NVRTC-specialised kernels run tiles of 12 qubits; "
                  "raise jit_max_kernels or use tile_k <= 11)");
        return cudaErrorInvalidValue;
    }
}

} // namespace qsv
