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
#include "qsv_internal.h"

#include <algorithm>

namespace qsv {

namespace {

constexpr int kNumBuf = 3;

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(a),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes,
                                          uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem_dst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void bulk_store(void* gdst, const void* smem_src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
                 "r"(smem_u32(smem_src)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

__device__ __forceinline__ void bulk_wait_read_all() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// ---------------------------------------------------------------- arithmetic
__device__ __forceinline__ void cmac(double2& acc, const double2 m, const double2 v) {
    acc.x = fma(m.x, v.x, acc.x);
    acc.x = fma(-m.y, v.y, acc.x);
    acc.y = fma(m.x, v.y, acc.y);
    acc.y = fma(m.y, v.x, acc.y);
}

__device__ __forceinline__ double2 cmul(const double2 a, const double2 b) {
    double2 r;
    r.x = fma(a.x, b.x, -a.y * b.y);
    r.y = fma(a.x, b.y, a.y * b.x);
    return r;
}

// Insert a zero bit at each of the ascending positions fixpos[0..nfix).
__device__ __forceinline__ uint32_t deposit(uint32_t g, const int8_t* fixpos, int nfix) {
    for (int i = 0; i < nfix; ++i) {
        const uint32_t p = static_cast<uint32_t>(fixpos[i]);
        const uint32_t lo = g & ((1u << p) - 1u);
        g = ((g ^ lo) << 1) | lo;
    }
    return g;
}

// ---------------------------------------------------------------- ops
template <int KK>
__device__ __forceinline__ void dense_rows(double2* tile, const double2* M, const uint32_t* off,
                                           uint32_t b, const double2 (&v)[1 << KK], int r0,
                                           int nrows) {
    constexpr int D = 1 << KK;
    // Two rows per iteration: four independent DFMA chains per thread.
#pragma unroll 1
    for (int r = r0; r < r0 + nrows; r += 2) {
        const double2* row0 = M + r * D;
        const double2* row1 = row0 + D;
        double2 a0 = make_double2(0.0, 0.0), a1 = make_double2(0.0, 0.0);
#pragma unroll
        for (int j = 0; j < D; ++j) {
            cmac(a0, row0[j], v[j]);
            cmac(a1, row1[j], v[j]);
        }
        tile[b | off[r]] = a0;
        tile[b | off[r + 1]] = a1;
    }
}

template <int KK, int K, int NT>
__device__ __forceinline__ void dense_op(double2* tile, const TileOp& op, const unsigned char* blob) {
    constexpr int D = 1 << KK;
    const int nfix = op.nfix;
    const uint32_t tctrl = op.tctrl;
    const uint32_t groups = 1u << (K - nfix);
    const double2* M = reinterpret_cast<const double2*>(blob + op.mat_byte);
    const uint32_t* off = reinterpret_cast<const uint32_t*>(blob + op.off_byte);
    if (groups >= static_cast<uint32_t>(NT)) {
        // One thread owns whole groups: read all 2^k members, then overwrite them.
#pragma unroll 1
        for (uint32_t g = threadIdx.x; g < groups; g += NT) {
            const uint32_t b = deposit(g, op.fixpos, nfix) | tctrl;
            double2 v[D];
#pragma unroll
            for (int j = 0; j < D; ++j)
                v[j] = tile[b | off[j]];
            dense_rows<KK>(tile, M, off, b, v, 0, D);
        }
    } else {
        // Fewer groups than threads: R threads share a group, each computing
        // D/R (>= 2) output rows.  All inputs are read before any output is written.
        const int R = min(NT / static_cast<int>(groups), D / 2);
        const int rows = D / R;
        const int t = threadIdx.x;
        const bool active = t < static_cast<int>(groups) * R;
        const uint32_t g = static_cast<uint32_t>(t) % groups;
        const int rb = t / static_cast<int>(groups);
        double2 v[D];
        uint32_t b = 0;
        if (active) {
            b = deposit(g, op.fixpos, nfix) | tctrl;
#pragma unroll
            for (int j = 0; j < D; ++j)
                v[j] = tile[b | off[j]];
        }
        __syncthreads();
        if (active)
            dense_rows<KK>(tile, M, off, b, v, rb * rows, rows);
    }
}

template <int K, int NT>
__device__ __forceinline__ void xperm_op(double2* tile, const TileOp& op) {
    const int nfix = op.nfix;
    const uint32_t tctrl = op.tctrl;
    const uint32_t groups = 1u << (K - nfix);
    const uint32_t tb = 1u << op.tpos[0];
    for (uint32_t g = threadIdx.x; g < groups; g += NT) {
        const uint32_t b = deposit(g, op.fixpos, nfix) | tctrl;
        const double2 a0 = tile[b];
        const double2 a1 = tile[b | tb];
        tile[b] = a1;
        tile[b | tb] = a0;
    }
}

template <int K, int NT>
__device__ __forceinline__ void diag_op(double2* tile, const TileOp& op, const unsigned char* blob,
                                        uint64_t full_base) {
    const int nfix = op.nfix;
    const uint32_t tctrl = op.tctrl;
    const uint32_t groups = 1u << (K - nfix);
    const int k = op.k;
    const int nin = op.nin;
    const uint32_t tmask = op.tmask;
    const double2* Dg = reinterpret_cast<const double2*>(blob + op.mat_byte);
    uint32_t e0 = 0;
    for (int j = nin; j < k; ++j)
        e0 |= static_cast<uint32_t>((full_base >> op.xbit[j - nin]) & 1ull) << j;
    if (nin == 0) {
        const double2 d = Dg[e0];
        for (uint32_t g = threadIdx.x; g < groups; g += NT) {
            const uint32_t idx = deposit(g, op.fixpos, nfix) | tctrl;
            tile[idx] = cmul(d, tile[idx]);
        }
        return;
    }
    for (uint32_t g = threadIdx.x; g < groups; g += NT) {
        const uint32_t idx = deposit(g, op.fixpos, nfix) | tctrl;
        uint32_t e = e0, m = tmask;
        for (int i = 0; m; ++i) {
            const int p = __ffs(m) - 1;
            e |= ((idx >> p) & 1u) << i;
            m &= m - 1;
        }
        tile[idx] = cmul(Dg[e], tile[idx]);
    }
}

struct GeomArg {
    int32_t L, nhigh;
    int32_t high[QSV_MAX_HIGH];
};

__device__ __forceinline__ uint64_t tile_base(uint64_t t, const GeomArg& g) {
    uint64_t base = t << g.L;
    for (int i = 0; i < g.nhigh; ++i) {
        const int h = g.high[i];
        const uint64_t lo = base & ((1ull << h) - 1ull);
        base = ((base ^ lo) << 1) | lo;
    }
    return base;
}

template <int K, int KMAX, int NT>
__global__ void __launch_bounds__(NT, 1)
pass_kernel(double2* __restrict__ psi, const unsigned char* __restrict__ gblob, uint32_t blob_bytes,
            int nops, const __grid_constant__ GeomArg geom, uint64_t rank_base, uint64_t ntiles) {
    constexpr int TILE = 1 << K;
    extern __shared__ __align__(128) unsigned char smem[];
    double2* bufs = reinterpret_cast<double2*>(smem);
    unsigned char* blob = smem + sizeof(double2) * kNumBuf * TILE;
    __shared__ uint64_t hi_off[1 << QSV_MAX_HIGH];
    __shared__ __align__(8) uint64_t mbar[kNumBuf];

    const int nh = 1 << geom.nhigh;
    const int L = geom.L;
    const uint32_t run_bytes = static_cast<uint32_t>(sizeof(double2)) << L;
    for (int j = threadIdx.x; j < nh; j += NT) {
        uint64_t o = 0;
        for (int i = 0; i < geom.nhigh; ++i)
            o |= static_cast<uint64_t>((j >> i) & 1) << geom.high[i];
        hi_off[j] = o;
    }
    {
        const int4* src = reinterpret_cast<const int4*>(gblob);
        int4* dst = reinterpret_cast<int4*>(blob);
        for (uint32_t i = threadIdx.x; i < blob_bytes / 16; i += NT)
            dst[i] = __ldg(src + i);
    }
    if (threadIdx.x == 0) {
        for (int b = 0; b < kNumBuf; ++b)
            mbar_init(&mbar[b], 1);
        fence_mbar_init();
    }
    __syncthreads();

    const uint64_t stride = gridDim.x;
    auto issue_load = [&](uint64_t t, int b) {
        const uint64_t base = tile_base(t, geom);
        double2* dst = bufs + b * TILE;
        mbar_expect_tx(&mbar[b], static_cast<uint32_t>(sizeof(double2) * TILE));
        for (int j = 0; j < nh; ++j)
            bulk_load(dst + (j << L), psi + base + hi_off[j], run_bytes, &mbar[b]);
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < kNumBuf - 1; ++s) {
            const uint64_t t = blockIdx.x + s * stride;
            if (t < ntiles)
                issue_load(t, s);
        }
    }

    const TileOp* ops = reinterpret_cast<const TileOp*>(blob);
    int it = 0;
    for (uint64_t t = blockIdx.x; t < ntiles; t += stride, ++it) {
        const int b = it % kNumBuf;
        if (threadIdx.x == 0) {
            const uint64_t tn = t + (kNumBuf - 1) * stride;
            if (tn < ntiles) {
                // Buffer (it + NBUF - 1) % NBUF was last stored from in iteration it - 1.
                bulk_wait_read_all();
                issue_load(tn, (it + kNumBuf - 1) % kNumBuf);
            }
        }
        mbar_wait(&mbar[b], static_cast<uint32_t>((it / kNumBuf) & 1));
        double2* tile = bufs + b * TILE;
        const uint64_t base = tile_base(t, geom);
        const uint64_t full_base = rank_base | base;

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
                if constexpr (KMAX >= 5 && K >= 5) { if (kk == 5) dense_op<5, K, NT>(tile, op, blob); }
            } else if (op.kind == QSV_OP_DIAG) {
                diag_op<K, NT>(tile, op, blob, full_base);
            } else {
                xperm_op<K, NT>(tile, op);
            }
        }
        // Make this thread's generic-proxy SMEM writes visible to the bulk-copy
        // (async) proxy, then let thread 0 stream the tile back.
        fence_proxy_async();
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int j = 0; j < nh; ++j)
                bulk_store(psi + base + hi_off[j], tile + (j << L), run_bytes);
            bulk_commit();
        }
    }
    if (threadIdx.x == 0)
        bulk_wait_all();
}

template <int K>
constexpr int threads_for() {
    return K >= 8 ? 256 : (K >= 6 ? 64 : 32);
}

template <int K, int KMAX>
cudaError_t launch_variant(const qsv_state* st, const Step& step, const unsigned char* d_blob,
                           uint64_t rank_base, cudaStream_t stream) {
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
    const uint64_t tiles = st->size >> K;
    const uint64_t grid = std::min<uint64_t>(tiles, static_cast<uint64_t>(per_sm) * sm_count);
    kern<<<static_cast<unsigned>(grid), NT, smem, stream>>>(st->amps, d_blob, step.blob_bytes,
                                                           step.nops, ga, rank_base, tiles);
    return cudaGetLastError();
}

template <int K>
cudaError_t launch_k(const qsv_state* st, const Step& step, const unsigned char* d_blob,
                     uint64_t rank_base, cudaStream_t stream) {
    if constexpr (K >= 9) {
        switch (step.geom.kmax <= 1 ? 1 : step.geom.kmax) {
        case 1: return launch_variant<K, 1>(st, step, d_blob, rank_base, stream);
        case 2: return launch_variant<K, 2>(st, step, d_blob, rank_base, stream);
        case 3: return launch_variant<K, 3>(st, step, d_blob, rank_base, stream);
        case 4: return launch_variant<K, 4>(st, step, d_blob, rank_base, stream);
        default: return launch_variant<K, 5>(st, step, d_blob, rank_base, stream);
        }
    } else {
        constexpr int KM = K < 5 ? K : 5;
        return launch_variant<K, KM>(st, step, d_blob, rank_base, stream);
    }
}

} // namespace

cudaError_t launch_pass(const qsv_state* st, const Step& step, const unsigned char* d_blob,
                        uint64_t rank_base, cudaStream_t stream) {
    switch (step.geom.K) {
    case 1: return launch_k<1>(st, step, d_blob, rank_base, stream);
    case 2: return launch_k<2>(st, step, d_blob, rank_base, stream);
    case 3: return launch_k<3>(st, step, d_blob, rank_base, stream);
    case 4: return launch_k<4>(st, step, d_blob, rank_base, stream);
    case 5: return launch_k<5>(st, step, d_blob, rank_base, stream);
    case 6: return launch_k<6>(st, step, d_blob, rank_base, stream);
    case 7: return launch_k<7>(st, step, d_blob, rank_base, stream);
    case 8: return launch_k<8>(st, step, d_blob, rank_base, stream);
    case 9: return launch_k<9>(st, step, d_blob, rank_base, stream);
    case 10: return launch_k<10>(st, step, d_blob, rank_base, stream);
    case 11: return launch_k<11>(st, step, d_blob, rank_base, stream);
    default: return cudaErrorInvalidValue;
    }
}

} // namespace qsv
