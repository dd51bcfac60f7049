// Device code of the fused multi-block pass (sm_100a), shared by the nvcc-built
// interpreter kernel (pass_kernel.cu) and the NVRTC-specialised kernels (jit.cu).
// See pass_kernel.cu for the design notes.  NVRTC-safe: no host headers.
#pragma once

#include "device_types.h"

namespace qsv {

// Thread index within the tile's thread group: a multi-tile CTA (pass_pipeline MT > 1)
// runs MT groups of NT threads, each on its own tile, in lockstep (the per-op CTA
// barriers keep every group at the same point of the straight-line pass code, so
// the warps a scheduler interleaves fetch the same instructions).  Every op body is
// written for one group of NT threads (NT is a power of two and a template
// parameter wherever this is used).
#define QSV_LTID (threadIdx.x & static_cast<unsigned>(NT - 1))


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

// Tensor-map tile copies of rank 1..5 (the instruction's dimensionality must match the
// map's rank; coordinates in elements, dim 0 counts doubles).
__device__ __forceinline__ void tensor_load(int rank, void* smem_dst, const TmaDesc* tmap, const int32_t (&c)[5],
                                            uint64_t* bar) {
    const uint32_t d = smem_u32(smem_dst), m = smem_u32(bar);
    const uint64_t t = reinterpret_cast<uint64_t>(tmap);
    switch (rank) {
    case 1:
        asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];"
                     ::"r"(d), "l"(t), "r"(c[0]), "r"(m) : "memory");
        break;
    case 2:
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(d), "l"(t), "r"(c[0]), "r"(c[1]), "r"(m) : "memory");
        break;
    case 3:
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                     ::"r"(d), "l"(t), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(m) : "memory");
        break;
    case 4:
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                     ::"r"(d), "l"(t), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(m) : "memory");
        break;
    default:
        asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                     ::"r"(d), "l"(t), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(m) : "memory");
        break;
    }
}

__device__ __forceinline__ void tensor_store(int rank, const TmaDesc* tmap, const int32_t (&c)[5], const void* smem_src) {
    const uint32_t sp = smem_u32(smem_src);
    const uint64_t t = reinterpret_cast<uint64_t>(tmap);
    switch (rank) {
    case 1:
        asm volatile("cp.async.bulk.tensor.1d.global.shared::cta.tile.bulk_group [%0, {%1}], [%2];" ::"l"(t), "r"(c[0]),
                     "r"(sp) : "memory");
        break;
    case 2:
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(t),
                     "r"(c[0]), "r"(c[1]), "r"(sp) : "memory");
        break;
    case 3:
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(t),
                     "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(sp) : "memory");
        break;
    case 4:
        asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(t),
                     "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(sp) : "memory");
        break;
    default:
        asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(t),
                     "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(sp) : "memory");
        break;
    }
}

__device__ __forceinline__ void bulk_wait_read_all() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// Wait until at most N of this thread's bulk groups are still reading SMEM.
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
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

// Groups of an op are enumerated directly in "deposited" form: with F the
// mask of the op's fixed tile bits (targets + tile controls), the successor of
// b = deposit(g) after a stride s is ((b | F) + deposit(s)) & ~F — the fixed
// bits, forced to 1, carry the addition across themselves.  Three integer ops
// per group instead of a loop over the fixed positions.
__device__ __forceinline__ uint32_t next_group(uint32_t b, uint32_t F, uint32_t dstride) {
    return ((b | F) + dstride) & ~F;
}

// ---------------------------------------------------------------- ops
// Warp-level complex mat-vec for k <= 4 (D = 2^k <= 16).  LPG = D*S lanes
// cooperate on one 2^k-amplitude group: lane (r, s) keeps columns
// [s*D/S, (s+1)*D/S) of matrix row r in registers for the whole op, reads the
// group members as SMEM broadcasts, and the S partial sums of a row are
// combined with warp shuffles.  A warp processes 32/LPG groups per step, so
// registers stay ~8*D/S per lane and no CTA barrier is needed inside the op
// (only __syncwarp between the reads and the in-place writes of a group).
template <int KK, int K, int NT>
__device__ __forceinline__ void dense_op(double2* tile, const TileOp& op, const unsigned char* blob) {
    constexpr int D = 1 << KK;
    constexpr int S = D >= 8 ? 2 : 1;     // column splits
    constexpr int LPG = D * S;            // lanes per group
    constexpr int GPW = 32 / LPG;         // groups per warp step
    constexpr int CPL = D / S;            // columns per lane
    constexpr int NW = NT / 32;
    constexpr uint32_t PER_STEP = NW * GPW;
    const int lane = QSV_LTID & 31;
    const int warp = QSV_LTID >> 5;
    const int sub = lane / LPG;
    const int r = (lane % LPG) / S;
    const int sp = (lane % LPG) % S;
    const double2* M = reinterpret_cast<const double2*>(blob + op.mat_byte);
    const uint32_t* off = reinterpret_cast<const uint32_t*>(blob + op.off_byte);
    double2 m[CPL];
    uint32_t o[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        m[c] = M[r * D + sp * CPL + c];
        o[c] = off[sp * CPL + c];
    }
    const uint32_t my_off = off[r];
    const int nfix = op.nfix;
    const uint32_t tctrl = op.tctrl;
    const uint32_t F = op.fmask;
    const uint32_t groups = 1u << (K - nfix);
    const uint32_t g = static_cast<uint32_t>(warp * GPW + sub);
    uint32_t b = deposit(g, op.fixpos, nfix);
    const uint32_t dstep = deposit(PER_STEP, op.fixpos, nfix);
    const uint32_t steps = groups >= PER_STEP ? groups / PER_STEP : 1u;
    const bool act = g < groups;
#pragma unroll 1
    for (uint32_t st = 0; st < steps; ++st) {
        const uint32_t idx = b | tctrl;
        double2 acc = make_double2(0.0, 0.0);
        if (act) {
#pragma unroll
            for (int c = 0; c < CPL; ++c)
                cmac(acc, m[c], tile[idx | o[c]]);
        }
        if constexpr (S > 1) {
            acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 1);
            acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 1);
        }
        __syncwarp();
        if (act && sp == 0)
            tile[idx | my_off] = acc;
        b = next_group(b, F, dstep);
    }
}

// Pass relabel (planner-chosen, applied after the pass's ops): tile bit b of every
// amplitude index moves to tile bit relabel[b], an in-place permutation of the tile.
// Thread t, iteration j handles source index x = t | j << log2(NT) mapped through an
// XOR-linear basis built on the host (src columns at blob+mat_byte, the matching
// destination columns 16 entries later).  The first three columns are chosen so that
// the 8 lanes of a quarter-warp hit 8 distinct 16-B bank slots on both the gather and
// the scatter, so the permutation costs two conflict-free SMEM sweeps.
template <int K, int NT>
__device__ __forceinline__ void relabel_op(double2* __restrict__ tile, const TileOp& op,
                                           const unsigned char* blob) {
    constexpr int TILE = 1 << K;
    constexpr int TB = NT >= 256 ? 8 : (NT >= 128 ? 7 : (NT >= 64 ? 6 : 5));
    const uint16_t* col = reinterpret_cast<const uint16_t*>(blob + op.mat_byte);
    if constexpr (TILE >= NT) {
        constexpr int APT = TILE / NT;
        constexpr int IB = K - TB;
        uint32_t sb = 0, db = 0;
#pragma unroll
        for (int b = 0; b < TB; ++b)
            if ((QSV_LTID >> b) & 1u) {
                sb ^= col[b];
                db ^= col[16 + b];
            }
        uint32_t is[IB > 0 ? IB : 1], id[IB > 0 ? IB : 1];
#pragma unroll
        for (int b = 0; b < IB; ++b) {
            is[b] = col[TB + b];
            id[b] = col[16 + TB + b];
        }
        double2 v[APT];
#pragma unroll
        for (int j = 0; j < APT; ++j) {
            uint32_t x = sb;
#pragma unroll
            for (int b = 0; b < IB; ++b)
                if ((j >> b) & 1)
                    x ^= is[b];
            v[j] = tile[x];
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < APT; ++j) {
            uint32_t x = db;
#pragma unroll
            for (int b = 0; b < IB; ++b)
                if ((j >> b) & 1)
                    x ^= id[b];
            tile[x] = v[j];
        }
    } else {
        const bool on = QSV_LTID < TILE;
        uint32_t sb = 0, db = 0;
#pragma unroll
        for (int b = 0; b < K; ++b)
            if ((QSV_LTID >> b) & 1u) {
                sb ^= col[b];
                db ^= col[16 + b];
            }
        double2 v0 = make_double2(0.0, 0.0);
        if (on)
            v0 = tile[sb];
        __syncthreads();
        if (on)
            tile[db] = v0;
    }
}

template <int K, int NT>
__device__ __forceinline__ void xperm_op(double2* tile, const TileOp& op) {
    const int nfix = op.nfix;
    const uint32_t tctrl = op.tctrl;
    const uint32_t F = op.fmask;
    const uint32_t groups = 1u << (K - nfix);
    const uint32_t tb = 1u << op.tpos[0];
    if (QSV_LTID >= groups)
        return;
    uint32_t b = deposit(QSV_LTID, op.fixpos, nfix);
    const uint32_t dstep = deposit(NT, op.fixpos, nfix);
    const uint32_t steps = groups >= static_cast<uint32_t>(NT) ? groups / NT : 1u;
#pragma unroll 2
    for (uint32_t st = 0; st < steps; ++st) {
        const uint32_t idx = b | tctrl;
        const double2 a0 = tile[idx];
        const double2 a1 = tile[idx | tb];
        tile[idx] = a1;
        tile[idx | tb] = a0;
        b = next_group(b, F, dstep);
    }
}

template <int K, int NT>
__device__ __forceinline__ void diag_op(double2* tile, const TileOp& op, const unsigned char* blob,
                                        uint64_t full_base) {
    const int nfix = op.nfix;
    const uint32_t tctrl = op.tctrl;
    const uint32_t F = op.fmask;
    const uint32_t groups = 1u << (K - nfix);
    const int k = op.k;
    const int nin = op.nin;
    const double2* Dg = reinterpret_cast<const double2*>(blob + op.mat_byte);
    uint32_t e0 = 0;
    for (int j = nin; j < k; ++j)
        e0 |= static_cast<uint32_t>((full_base >> op.xbit[j - nin]) & 1ull) << j;
    if (QSV_LTID >= groups)
        return;
    uint32_t b = deposit(QSV_LTID, op.fixpos, nfix);
    const uint32_t dstep = deposit(NT, op.fixpos, nfix);
    const uint32_t steps = groups >= static_cast<uint32_t>(NT) ? groups / NT : 1u;
    if (nin == 0) {
        const double2 d = Dg[e0];
#pragma unroll 4
        for (uint32_t st = 0; st < steps; ++st) {
            const uint32_t idx = b | tctrl;
            tile[idx] = cmul(d, tile[idx]);
            b = next_group(b, F, dstep);
        }
    } else if (nin == 1) {
        const int p = __ffs(op.tmask) - 1;
        const double2 d0 = Dg[e0], d1 = Dg[e0 | 1u];
#pragma unroll 4
        for (uint32_t st = 0; st < steps; ++st) {
            const uint32_t idx = b | tctrl;
            tile[idx] = cmul(((idx >> p) & 1u) ? d1 : d0, tile[idx]);
            b = next_group(b, F, dstep);
        }
    } else {
        const uint8_t* plo = blob + op.ptab_byte;
        const uint8_t* phi = plo + 32;
#pragma unroll 2
        for (uint32_t st = 0; st < steps; ++st) {
            const uint32_t idx = b | tctrl;
            const uint32_t e = e0 | plo[idx & 31u] | phi[idx >> 5];
            tile[idx] = cmul(Dg[e], tile[idx]);
            b = next_group(b, F, dstep);
        }
    }
}

// k = 5 (D = 32): one thread per group, all 32 members in registers.
template <int K, int NT>
__device__ __forceinline__ void dense5_op(double2* tile, const TileOp& op, const unsigned char* blob) {
    constexpr int D = 32;
    const int nfix = op.nfix;
    const uint32_t tctrl = op.tctrl;
    const uint32_t groups = 1u << (K - nfix);
    const double2* M = reinterpret_cast<const double2*>(blob + op.mat_byte);
    const uint32_t* off = reinterpret_cast<const uint32_t*>(blob + op.off_byte);
    const bool many = groups >= static_cast<uint32_t>(NT);
    const int R = many ? 1 : min(NT / static_cast<int>(groups), D);
    const int rows = D / R;
#pragma unroll 1
    for (uint32_t base_t = 0; base_t < (many ? groups : 1u); base_t += NT) {
        const int t = static_cast<int>(QSV_LTID);
        const uint32_t g = many ? base_t + t : static_cast<uint32_t>(t) % groups;
        const int rb = many ? 0 : t / static_cast<int>(groups);
        const bool act = many ? g < groups : t < static_cast<int>(groups) * R;
        double2 v[D];
        uint32_t b = 0;
        if (act) {
            b = deposit(g, op.fixpos, nfix) | tctrl;
#pragma unroll
            for (int j = 0; j < D; ++j)
                v[j] = tile[b | off[j]];
        }
        if (!many)
            __syncthreads();
        if (act) {
#pragma unroll 1
            for (int rr = 0; rr < rows; ++rr) {
                const int row = rb * rows + rr;
                double2 acc = make_double2(0.0, 0.0);
#pragma unroll
                for (int j = 0; j < D; ++j)
                    cmac(acc, M[row * D + j], v[j]);
                tile[b | off[row]] = acc;
            }
        }
    }
}

// ---------------------------------------------------------------- DMMA16
// Dense 16x16 complex unitary on 4 tile qubits with the FP64 tensor cores.  The
// complex mat-vec of every group is one column of a real GEMM
//     [Yr; Yi] (32 x G) = [[Mr, -Mi], [Mi, Mr]] (32 x 32) . [Xr; Xi] (32 x G)
// cut into mma.sync.m8n8k4.f64 tiles: 4 row blocks (Re members 0-7, 8-15, Im 0-7,
// 8-15) x 8 k-steps (Re members 0-3, ..., Im members 12-15) per 8 groups.  A warp
// owns whole 8-group column blocks, so no CTA barrier is needed inside the op: its
// lanes read the groups (LDS.128 = the Re and Im rows of one member), the MMAs
// consume every lane's fragment, then the lanes write the results back (STS.128
// pairs the Re and Im accumulators of one member).  Per amplitude: 64 DMMA MACs
// (128 flop, the dense cost) issued as 1/4 instruction instead of ~50 DFMA/DMUL.
// Fragment layout (PTX m8n8k4 .f64): A[g][t], B[t][g], C[g][2t + i] for lane = 4g + t.
__device__ __forceinline__ void dmma_m8n8k4(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

template <int K, int NT>
__device__ __forceinline__ void dmma16_op(double2* tile, const TileOp& op, const unsigned char* blob) {
    constexpr int NW = NT / 32;
    const uint32_t lane = QSV_LTID & 31u;
    const uint32_t warp = QSV_LTID >> 5;
    const uint32_t g = lane >> 2, t = lane & 3u;
    const uint32_t groups = 1u << (K - op.nfix);
    const uint32_t nblk = (groups + 7u) >> 3;  // 8-group column blocks
    if (warp >= nblk)
        return;
    const double2* M = reinterpret_cast<const double2*>(blob + op.mat_byte);
    // A fragments: M[8 mt + g][4 ks + t] for mt < 2, ks < 4 (Re and Im parts; -Im once)
    double ar[2][4], ai[2][4], an[2][4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
            const double2 m = M[(8 * mt + g) * 16 + 4 * ks + t];
            ar[mt][ks] = m.x;
            ai[mt][ks] = m.y;
            an[mt][ks] = -m.y;
        }
    // member offsets: B reads members 4q + t, D writes members 8h + g
    const uint32_t m0 = 1u << op.tpos[0], m1 = 1u << op.tpos[1], m2 = 1u << op.tpos[2], m3 = 1u << op.tpos[3];
    auto moff = [&](uint32_t j) {
        return ((j & 1u) ? m0 : 0u) | ((j & 2u) ? m1 : 0u) | ((j & 4u) ? m2 : 0u) | ((j & 8u) ? m3 : 0u);
    };
    uint32_t ob[4], od[2];
#pragma unroll
    for (int q = 0; q < 4; ++q)
        ob[q] = moff(4u * q + t);
#pragma unroll
    for (int h = 0; h < 2; ++h)
        od[h] = moff(8u * h + g);
    const uint32_t tctrl = op.tctrl;
#pragma unroll 1
    for (uint32_t blk = warp; blk < nblk; blk += NW) {
        const uint32_t gb = blk * 8u + g;  // this lane's B column (group)
        const bool vb = gb < groups;
        const uint32_t bb = vb ? (deposit(gb, op.fixpos, op.nfix) | tctrl) : 0u;
        double xr[4], xi[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double2 x = vb ? tile[bb | ob[q]] : make_double2(0.0, 0.0);
            xr[q] = x.x;
            xi[q] = x.y;
        }
        double d[4][2];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
            d[mt][0] = d[mt][1] = 0.0;
        // k-outer so the four row-block accumulations are independent chains
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
            const double b = ks < 4 ? xr[ks] : xi[ks - 4];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
                const int r = mt & 1, kk = ks & 3;
                const double a = mt < 2 ? (ks < 4 ? ar[r][kk] : an[r][kk]) : (ks < 4 ? ai[r][kk] : ar[r][kk]);
                dmma_m8n8k4(d[mt][0], d[mt][1], a, b);
            }
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const uint32_t gd = blk * 8u + 2u * t + static_cast<uint32_t>(i);
            if (gd < groups) {
                const uint32_t bd = deposit(gd, op.fixpos, op.nfix) | tctrl;
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    tile[bd | od[h]] = make_double2(d[h][i], d[h + 2][i]);
            }
        }
    }
}

// ---------------------------------------------------------------- RBLOCK
// A register block holds one group of NV = 2^KB amplitudes (KB = 3 or 4 block
// qubits) per thread and applies a list of native gates to it in registers;
// the list is uniform over the CTA, so the per-primitive switch is a uniform
// branch.  Register v[j] holds group member j ^ r, where r is this lane's
// member rotation (it spreads the lanes of a quarter-warp over the SMEM
// banks); the host stores every matrix in its rotated variants.
template <int NV, int Q>
__device__ __forceinline__ void rb_u1(double2 (&v)[NV], const double2* U) {
    const double2 u00 = U[0], u01 = U[1], u10 = U[2], u11 = U[3];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        if (j & (1 << Q))
            continue;
        const double2 x0 = v[j], x1 = v[j | (1 << Q)];
        double2 r0 = make_double2(0.0, 0.0), r1 = make_double2(0.0, 0.0);
        cmac(r0, u00, x0);
        cmac(r0, u01, x1);
        cmac(r1, u10, x0);
        cmac(r1, u11, x1);
        v[j] = r0;
        v[j | (1 << Q)] = r1;
    }
}

// Real 2x2 (H, RY, products of them): the real and imaginary parts of the
// amplitudes are transformed independently, 4 DFMA per amplitude.
template <int NV, int Q>
__device__ __forceinline__ void rb_u1r(double2 (&v)[NV], const double2* U) {
    const double u00 = U[0].x, u01 = U[1].x, u10 = U[2].x, u11 = U[3].x;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        if (j & (1 << Q))
            continue;
        const double2 x0 = v[j], x1 = v[j | (1 << Q)];
        v[j] = make_double2(fma(u00, x0.x, u01 * x1.x), fma(u00, x0.y, u01 * x1.y));
        v[j | (1 << Q)] = make_double2(fma(u10, x0.x, u11 * x1.x), fma(u10, x0.y, u11 * x1.y));
    }
}

// Real diagonal, imaginary off-diagonal 2x2 (RX): [[c0, i s01], [i s10, c1]].
template <int NV, int Q>
__device__ __forceinline__ void rb_u1i(double2 (&v)[NV], const double2* U) {
    const double c0 = U[0].x, s01 = U[1].y, s10 = U[2].y, c1 = U[3].x;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        if (j & (1 << Q))
            continue;
        const double2 x0 = v[j], x1 = v[j | (1 << Q)];
        v[j] = make_double2(fma(c0, x0.x, -s01 * x1.y), fma(c0, x0.y, s01 * x1.x));
        v[j | (1 << Q)] = make_double2(fma(c1, x1.x, -s10 * x0.y), fma(c1, x1.y, s10 * x0.x));
    }
}

template <int NV, int A, int B>  // A < B: matrix bit 0 <-> block qubit A, bit 1 <-> B
__device__ __forceinline__ void rb_u2(double2 (&v)[NV], const double2* M) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        if (j & ((1 << A) | (1 << B)))
            continue;
        const int i1 = j | (1 << A), i2 = j | (1 << B), i3 = j | (1 << A) | (1 << B);
        const double2 x0 = v[j], x1 = v[i1], x2 = v[i2], x3 = v[i3];
        double2 y[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            double2 acc = make_double2(0.0, 0.0);
            cmac(acc, M[4 * r + 0], x0);
            cmac(acc, M[4 * r + 1], x1);
            cmac(acc, M[4 * r + 2], x2);
            cmac(acc, M[4 * r + 3], x3);
            y[r] = acc;
        }
        v[j] = y[0];
        v[i1] = y[1];
        v[i2] = y[2];
        v[i3] = y[3];
    }
}

// CX on (C, T) swaps members with bit C = 1, i.e. registers whose bit C
// differs from the rotation bit r_C.
template <int NV, int C, int T>
__device__ __forceinline__ void rb_cx(double2 (&v)[NV], uint32_t r) {
    const bool rc = (r >> C) & 1u;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        if (j & (1 << T))
            continue;
        const bool fire = (((j >> C) & 1) != 0) != rc;
        const double2 x0 = v[j], x1 = v[j | (1 << T)];
        v[j] = fire ? x1 : x0;
        v[j | (1 << T)] = fire ? x0 : x1;
    }
}

template <int NV>
__device__ __forceinline__ void rb_diag(double2 (&v)[NV], const double2* D, uint32_t r) {
#pragma unroll
    for (int j = 0; j < NV; ++j)
        v[j] = cmul(D[j ^ r], v[j]);
}

#define RB_CODE(kind, a, b) (((kind) << 4) | ((a) << 2) | (b))

template <int NV>
__device__ __forceinline__ void rb_apply(double2 (&v)[NV], const DevPrim pr, const double2* m, uint32_t r) {
    const uint32_t ra = (r >> pr.a) & 1u, rb = (r >> pr.b) & 1u;
    const double2* m1 = m + 4 * ra;                 // U1 variant (U or XUX)
    const double2* m2 = m + 16 * (ra | (rb << 1));  // U2 variant
    switch (RB_CODE(pr.kind, pr.a, pr.b)) {
    case RB_CODE(QSV_PRIM_U1, 0, 0): rb_u1<NV, 0>(v, m1); break;
    case RB_CODE(QSV_PRIM_U1, 1, 0): rb_u1<NV, 1>(v, m1); break;
    case RB_CODE(QSV_PRIM_U1, 2, 0): rb_u1<NV, 2>(v, m1); break;
    case RB_CODE(QSV_PRIM_U1R, 0, 0): rb_u1r<NV, 0>(v, m1); break;
    case RB_CODE(QSV_PRIM_U1R, 1, 0): rb_u1r<NV, 1>(v, m1); break;
    case RB_CODE(QSV_PRIM_U1R, 2, 0): rb_u1r<NV, 2>(v, m1); break;
    case RB_CODE(QSV_PRIM_U1I, 0, 0): rb_u1i<NV, 0>(v, m1); break;
    case RB_CODE(QSV_PRIM_U1I, 1, 0): rb_u1i<NV, 1>(v, m1); break;
    case RB_CODE(QSV_PRIM_U1I, 2, 0): rb_u1i<NV, 2>(v, m1); break;
    case RB_CODE(QSV_PRIM_U2, 0, 1): rb_u2<NV, 0, 1>(v, m2); break;
    case RB_CODE(QSV_PRIM_U2, 0, 2): rb_u2<NV, 0, 2>(v, m2); break;
    case RB_CODE(QSV_PRIM_U2, 1, 2): rb_u2<NV, 1, 2>(v, m2); break;
    case RB_CODE(QSV_PRIM_CX, 0, 1): rb_cx<NV, 0, 1>(v, r); break;
    case RB_CODE(QSV_PRIM_CX, 0, 2): rb_cx<NV, 0, 2>(v, r); break;
    case RB_CODE(QSV_PRIM_CX, 1, 0): rb_cx<NV, 1, 0>(v, r); break;
    case RB_CODE(QSV_PRIM_CX, 1, 2): rb_cx<NV, 1, 2>(v, r); break;
    case RB_CODE(QSV_PRIM_CX, 2, 0): rb_cx<NV, 2, 0>(v, r); break;
    case RB_CODE(QSV_PRIM_CX, 2, 1): rb_cx<NV, 2, 1>(v, r); break;
    default:
        if constexpr (NV == 16) {
            switch (RB_CODE(pr.kind, pr.a, pr.b)) {
            case RB_CODE(QSV_PRIM_U1, 3, 0): rb_u1<NV, 3>(v, m1); return;
            case RB_CODE(QSV_PRIM_U1R, 3, 0): rb_u1r<NV, 3>(v, m1); return;
            case RB_CODE(QSV_PRIM_U1I, 3, 0): rb_u1i<NV, 3>(v, m1); return;
            case RB_CODE(QSV_PRIM_U2, 0, 3): rb_u2<NV, 0, 3>(v, m2); return;
            case RB_CODE(QSV_PRIM_U2, 1, 3): rb_u2<NV, 1, 3>(v, m2); return;
            case RB_CODE(QSV_PRIM_U2, 2, 3): rb_u2<NV, 2, 3>(v, m2); return;
            case RB_CODE(QSV_PRIM_CX, 0, 3): rb_cx<NV, 0, 3>(v, r); return;
            case RB_CODE(QSV_PRIM_CX, 1, 3): rb_cx<NV, 1, 3>(v, r); return;
            case RB_CODE(QSV_PRIM_CX, 2, 3): rb_cx<NV, 2, 3>(v, r); return;
            case RB_CODE(QSV_PRIM_CX, 3, 0): rb_cx<NV, 3, 0>(v, r); return;
            case RB_CODE(QSV_PRIM_CX, 3, 1): rb_cx<NV, 3, 1>(v, r); return;
            case RB_CODE(QSV_PRIM_CX, 3, 2): rb_cx<NV, 3, 2>(v, r); return;
            default: break;
            }
        }
        rb_diag<NV>(v, m, r);  // QSV_PRIM_DIAG16: 2^KB-entry diagonal
        break;
    }
}

template <int K, int NT, int KB>
__device__ __forceinline__ void rblock_op(double2* tile, const TileOp& op, const unsigned char* blob) {
    constexpr int NV = 1 << KB;
    uint32_t mk[KB];
#pragma unroll
    for (int i = 0; i < KB; ++i)
        mk[i] = 1u << op.tpos[i];
    const int nfix = op.nfix;
    const uint32_t tctrl = op.tctrl;
    const uint32_t F = op.fmask;
    const uint32_t groups = 1u << (K - nfix);
    if (QSV_LTID >= groups)
        return;
    // this lane's member rotation (bank spreading), as block bits and tile offset
    const uint32_t r = (op.rot_tab >> (4 * (QSV_LTID & 7))) & 15u;
    uint32_t offr = 0;
#pragma unroll
    for (int i = 0; i < KB; ++i)
        offr |= ((r >> i) & 1u) ? mk[i] : 0u;
    uint32_t b = deposit(QSV_LTID, op.fixpos, nfix);
    const uint32_t dstep = deposit(NT, op.fixpos, nfix);
    const uint32_t steps = groups >= static_cast<uint32_t>(NT) ? groups / NT : 1u;
    const DevPrim* prims = reinterpret_cast<const DevPrim*>(blob + op.prim_byte);
    const int np = op.nprim;
#pragma unroll 1
    for (uint32_t st = 0; st < steps; ++st) {
        const uint32_t base = b | tctrl | offr;
        double2 v[NV];
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            uint32_t o = 0;
#pragma unroll
            for (int i = 0; i < KB; ++i)
                o |= ((j >> i) & 1) ? mk[i] : 0u;
            v[j] = tile[base ^ o];
        }
#pragma unroll 1
        for (int p = 0; p < np; ++p) {
            const DevPrim pr = prims[p];
            rb_apply<NV>(v, pr, reinterpret_cast<const double2*>(blob + pr.data_byte), r);
        }
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            uint32_t o = 0;
#pragma unroll
            for (int i = 0; i < KB; ++i)
                o |= ((j >> i) & 1) ? mk[i] : 0u;
            tile[base ^ o] = v[j];
        }
        b = next_group(b, F, dstep);
    }
}

// ---------------------------------------------------------------- PARPHASE
// amp *= P[parity(index & mask)] for amplitudes with the controls set; the
// out-of-tile part of the parity is CTA-uniform.
template <int K, int NT>
__device__ __forceinline__ void parphase_op(double2* tile, const TileOp& op, const unsigned char* blob,
                                            uint64_t full_base) {
    const double2* P = reinterpret_cast<const double2*>(blob + op.mat_byte);
    const uint32_t ext = static_cast<uint32_t>(__popcll(full_base & op.xmask)) & 1u;
    const double2 p0 = P[ext], p1 = P[ext ^ 1u];
    const uint32_t tmask = op.tmask;
    const int nfix = op.nfix;
    const uint32_t tctrl = op.tctrl;
    const uint32_t F = op.fmask;
    const uint32_t groups = 1u << (K - nfix);
    if (QSV_LTID >= groups)
        return;
    uint32_t b = deposit(QSV_LTID, op.fixpos, nfix);
    const uint32_t dstep = deposit(NT, op.fixpos, nfix);
    const uint32_t steps = groups >= static_cast<uint32_t>(NT) ? groups / NT : 1u;
#pragma unroll 4
    for (uint32_t st = 0; st < steps; ++st) {
        const uint32_t idx = b | tctrl;
        tile[idx] = cmul((__popc(idx & tmask) & 1) ? p1 : p0, tile[idx]);
        b = next_group(b, F, dstep);
    }
}

// ------------------------------------------------ diagonal epilogue constants
// Per-tile (CTA-uniform) parts of the diagonal ops the JIT folds into the
// preceding register block (the per-amplitude parts are generated inline with
// the same arithmetic as diag_op / phaseprod_op / parphase_op).
__device__ __forceinline__ uint32_t diag_ext(const TileOp& op, uint64_t full_base) {
    uint32_t e0 = 0;
    for (int j = op.nin; j < op.k; ++j)
        e0 |= static_cast<uint32_t>((full_base >> op.xbit[j - op.nin]) & 1ull) << j;
    return e0;
}

__device__ __forceinline__ void par_consts(const TileOp& op, const unsigned char* blob, uint64_t full_base,
                                           double2& p0, double2& p1) {
    const double2* P = reinterpret_cast<const double2*>(blob + op.mat_byte);
    const uint32_t ext = static_cast<uint32_t>(__popcll(full_base & op.xmask)) & 1u;
    p0 = P[ext];
    p1 = P[ext ^ 1u];
}

__device__ __forceinline__ double2 pp_const(const TileOp& op, const unsigned char* blob, uint64_t full_base) {
    const double2* tab = reinterpret_cast<const double2*>(blob + op.mat_byte);
    const ExtFactor* ext = reinterpret_cast<const ExtFactor*>(blob + op.prim_byte);
    double2 c = tab[0];
    for (int i = 0; i < op.nprim; ++i)
        if ((full_base >> ext[i].bit) & 1ull)
            c = cmul(c, make_double2(ext[i].re, ext[i].im));
    return c;
}

// ---------------------------------------------------------------- PHASEPROD
// amp *= c * prod_{q in Q, bit q set} f_q for amplitudes with the controls set.
// In-tile factors are pre-tabulated over the low 5 tile bits (A[32]) and the
// high tile bits (B[64]); out-of-tile factors collapse into a CTA constant.
template <int K, int NT>
__device__ __forceinline__ void phaseprod_op(double2* tile, const TileOp& op, const unsigned char* blob,
                                             uint64_t full_base) {
    const double2* tab = reinterpret_cast<const double2*>(blob + op.mat_byte);
    const ExtFactor* ext = reinterpret_cast<const ExtFactor*>(blob + op.prim_byte);
    double2 c = tab[0];
    for (int i = 0; i < op.nprim; ++i)
        if ((full_base >> ext[i].bit) & 1ull)
            c = cmul(c, make_double2(ext[i].re, ext[i].im));
    const double2* A = tab + 1;
    const double2* B = tab + 33;
    const int nfix = op.nfix;
    const uint32_t tctrl = op.tctrl;
    const uint32_t F = op.fmask;
    const uint32_t groups = 1u << (K - nfix);
    if (QSV_LTID >= groups)
        return;
    uint32_t b = deposit(QSV_LTID, op.fixpos, nfix);
    const uint32_t dstep = deposit(NT, op.fixpos, nfix);
    const uint32_t steps = groups >= static_cast<uint32_t>(NT) ? groups / NT : 1u;
#pragma unroll 4
    for (uint32_t st = 0; st < steps; ++st) {
        const uint32_t idx = b | tctrl;
        const double2 w = cmul(c, cmul(A[idx & 31u], B[idx >> 5]));
        tile[idx] = cmul(w, tile[idx]);
        b = next_group(b, F, dstep);
    }
}

__device__ __forceinline__ uint64_t tile_base(uint64_t t, const GeomArg& g) {
    uint64_t base = t << g.L;
    // insert zeros at the high tile bits and the region bits, ascending
    int i = 0, j = 0;
    while (i < g.nhigh || j < g.nreg) {
        int h;
        if (j >= g.nreg || (i < g.nhigh && g.high[i] < g.reg[j]))
            h = g.high[i++];
        else
            h = g.reg[j++];
        const uint64_t lo = base & ((1ull << h) - 1ull);
        base = ((base ^ lo) << 1) | lo;
    }
    return base | g.rval;
}

// The persistent TMA pipeline of a pass; `ops(tile, blob, full_base)` applies
// the pass's ops to one SMEM-resident tile (interpreted or JIT-specialised).
// NBUF tile buffers, loads issued PD tiles ahead: the load of tile t + PD reuses
// the buffer of tile t + PD - NBUF, whose store was committed NBUF - PD - 1
// iterations before the current one, so warp 0 only waits for stores older than
// that (NBUF = 2, PD = 1: the previous tile's store must have left SMEM).
// SPREAD: every warp issues the TMA copies of its share of the runs (run j belongs to
// warp j % NW) and arms the mbarrier for those bytes (one arrival per warp), instead of
// warp 0 carrying all of it; each lane only ever waits for its own store groups, which
// read exactly the SMEM runs it reloads.  Warps then reach the per-op barriers together.
template <int K, int NT, int NBUF = kNumBuf, int PD = NBUF - 1, bool SPREAD = true, int MT = 1, typename Ops>
__device__ __forceinline__ void pass_pipeline(double2* __restrict__ psi, const unsigned char* __restrict__ gblob,
                                              uint32_t blob_bytes, const GeomArg& geom, uint64_t rank_base,
                                              uint64_t ntiles, Ops&& ops, const TmaDesc* tmap = nullptr) {
    // MT tile groups of NT threads per CTA (see QSV_LTID): group `sub` owns NBUF buffers
    // and mbarriers and processes tiles T * MT + sub of the CTA's tile sequence T.  All
    // groups run the same number of iterations (a group past the last tile still runs
    // the ops on its stale buffer, for the shared barriers, but neither loads nor stores).
    constexpr int TILE = 1 << K;
    extern __shared__ __align__(128) unsigned char smem[];
    static_assert(PD >= 1 && PD < NBUF, "prefetch distance must be in [1, NBUF)");
    static_assert(MT >= 1 && MT <= 4, "tile groups per CTA must be in [1, 4]");
    const int sub = MT > 1 ? static_cast<int>(threadIdx.x) / NT : 0;
    double2* bufs = reinterpret_cast<double2*>(smem) + static_cast<size_t>(sub) * NBUF * TILE;
    unsigned char* blob = smem + sizeof(double2) * MT * NBUF * TILE;
    __shared__ uint64_t hi_off[1 << QSV_MAX_HIGH];
    __shared__ __align__(8) uint64_t mbar_all[MT * NBUF];
    uint64_t* mbar = mbar_all + sub * NBUF;

    const int nh = 1 << geom.nhigh;
    const int L = geom.L;
    // High qubits that continue the low run (high[i] == L + i) are contiguous in
    // HBM too: merge them into the bulk copies (fewer, longer TMA runs).
    int m = 0;
    while (m < geom.nhigh && geom.high[m] == L + m && !(geom.peer && geom.sv_tile && geom.high[m] == geom.sv))
        ++m;  // (a fused swap's bit sv must separate runs: its two halves have different sources)
    const int RL = L + m;
    const int nruns = nh >> m;
    const uint32_t run_bytes = static_cast<uint32_t>(sizeof(double2)) << RL;
    for (int j = threadIdx.x; j < nh; j += NT * MT) {
        uint64_t o = 0;
        for (int i = 0; i < geom.nhigh; ++i)
            o |= static_cast<uint64_t>((j >> i) & 1) << geom.high[i];
        hi_off[j] = o;
    }
    {
        const int4* src = reinterpret_cast<const int4*>(gblob);
        int4* dst = reinterpret_cast<int4*>(blob);
        for (uint32_t i = threadIdx.x; i < blob_bytes / 16; i += NT * MT)
            dst[i] = __ldg(src + i);
    }
    // tensor-map mode: one thread issues a few box copies per tile instead of the warps
    // issuing one bulk copy per contiguous run
    const bool tens = tmap != nullptr && geom.tm_rank > 0;
    const int NW = tens ? 1 : (SPREAD ? NT / 32 : 1);  // warps of a group issuing TMA copies
    if (threadIdx.x == 0) {
        for (int b = 0; b < MT * NBUF; ++b)
            mbar_init(&mbar_all[b], NW);
        fence_mbar_init();
    }
    __syncthreads();

    const uint64_t stride = gridDim.x;
    // The issuing warps drive the TMA bulk engine: lane 0 of each arms the tile's
    // mbarrier with its byte count, then its lanes issue that warp's run copies.
    const int lane = threadIdx.x & 31;
    const int warp = static_cast<int>(QSV_LTID >> 5);
    const bool issuer = warp < NW;
    const int my_runs = nruns > warp ? (nruns - warp + NW - 1) / NW : 0;
    // fused swap: whole-tile mode pairs tile t on the ranks with sgbit = 0 with tile
    // t ^ (1 << sv_tidx) on their peers, so the twins of an iteration are partner tiles
    const bool fused = geom.peer != nullptr;
    const uint64_t txor = (fused && !geom.sv_tile && geom.sgbit) ? (1ull << geom.sv_tidx) : 0ull;
    const uint64_t svm = fused ? (1ull << geom.sv) : 0ull;
    const uint64_t sgm = fused && geom.sgbit ? svm : 0ull;
    auto tile_of = [&](uint64_t T) { return (T * MT + static_cast<uint64_t>(sub)) ^ txor; };
    // does this tile read (whole mode) or hold (mixed mode) data of the peer?
    auto remote_tile = [&](uint64_t base) { return fused && (geom.sv_tile || (base & svm) != sgm); };
    // tensor copies: coordinates of the box that holds tile base `bb` (+ iterated bits e)
    auto tm_coords = [&](uint64_t bb, int32_t (&c)[5]) {
#pragma unroll
        for (int d = 0; d < 5; ++d) {
            if (d >= geom.tm_rank) {
                c[d] = 0;
                continue;
            }
            const int lo = geom.tm_s[d];
            const uint64_t v = bb >> lo;
            const int hi = d + 1 < geom.tm_rank ? geom.tm_s[d + 1] : 63;
            c[d] = static_cast<int32_t>(v & ((1ull << (hi - lo)) - 1ull)) << (d == 0 ? 1 : 0);
        }
    };
    auto issue_load = [&](uint64_t t, int b) {
        const uint64_t base = tile_base(geom.tile0 + t, geom);
        double2* dst = bufs + b * TILE;
        if (tens) {
            if (geom.poison) {  // debug: NaN in the whole buffer before its tensor loads
                const double nan = __longlong_as_double(0x7ff8dead00000000ll);
                for (int e = lane; e < TILE; e += 32)
                    dst[e] = make_double2(nan, nan);
                fence_proxy_async();
                __syncwarp();
            }
            if (lane == 0) {
                mbar_expect_tx(&mbar[b], static_cast<uint32_t>(sizeof(double2) * TILE));
                for (int e = 0; e < (1 << geom.tm_nx); ++e) {
                    uint64_t bb = base;
                    for (int i = 0; i < geom.tm_nx; ++i)
                        bb |= static_cast<uint64_t>((e >> i) & 1) << geom.tm_x[i];
                    int32_t c[5];
                    tm_coords(bb, c);
                    tensor_load(geom.tm_rank, dst + static_cast<uint32_t>(e) * geom.tm_box_amps, tmap, c, &mbar[b]);
                }
            }
            return;
        }
        if (lane == 0)
            mbar_expect_tx(&mbar[b], static_cast<uint32_t>(my_runs) * run_bytes);
        __syncwarp();
        if (geom.poison) {  // debug: NaN in this warp's runs of the buffer, then the loads
            const double nan = __longlong_as_double(0x7ff8dead00000000ll);
            for (int k = 0; k < my_runs; ++k) {
                double2* run = dst + ((warp + NW * k) << RL);
                for (int e = lane; e < (1 << RL); e += 32)
                    run[e] = make_double2(nan, nan);
            }
            fence_proxy_async();
            __syncwarp();
        }
        for (int k = lane; k < my_runs; k += 32) {
            const int j = warp + NW * k;
            const uint64_t idx = base + hi_off[j << m];
            const double2* src = psi + idx;
            if (fused && !geom.spush && (idx & svm) != sgm)
                src = geom.peer + (idx ^ svm);  // NVLink: the peer's slot of this amplitude run
            bulk_load(dst + (j << RL), src, run_bytes, &mbar[b]);
        }
    };

    const uint64_t nT = (ntiles + MT - 1) / MT;  // CTA-level tile steps
    if (issuer) {
        for (int s = 0; s < PD; ++s) {
            const uint64_t t = tile_of(blockIdx.x + s * stride);
            if (blockIdx.x + s * stride < nT && t < ntiles)
                issue_load(t, s);
        }
    }

    int it = 0;
    for (uint64_t T = blockIdx.x; T < nT; T += stride, ++it) {
        const int b = it % NBUF;
        const uint64_t t = tile_of(T);
        const bool valid = t < ntiles;
        if (issuer) {
            const uint64_t Tn = T + PD * stride;
            const uint64_t tn = tile_of(Tn);
            if (Tn < nT && tn < ntiles) {
                // Buffer (it + PD) % NBUF was last stored from in iteration
                // it + PD - NBUF: every lane waits for its own store groups that old.
                bulk_wait_read<NBUF - PD - 1>();
                __syncwarp();
                issue_load(tn, (it + PD) % NBUF);
            }
        }
        if (valid)
            mbar_wait(&mbar[b], static_cast<uint32_t>((it / NBUF) & 1));
        double2* tile = bufs + b * TILE;
        const uint64_t base = valid ? tile_base(geom.tile0 + t, geom) : 0;
        const uint64_t full_base = rank_base | base;
        const bool remote = valid && remote_tile(base);
        const unsigned long long flag_val = (static_cast<unsigned long long>(geom.epoch) << 32) | (it + 1u);
        if (remote && threadIdx.x == 0)  // this CTA has read the peer's slots of the tile
            asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(geom.flag_peer + blockIdx.x), "l"(flag_val)
                         : "memory");
        if (MT > 1 && !valid && issuer)
            bulk_wait_read_all();  // the stale buffer may still feed a store; every op starts with a CTA barrier

        ops(tile, blob, full_base);
        // Make this thread's generic-proxy SMEM writes visible to the bulk-copy
        // (async) proxy, then let the issuing warps stream the tile back.
        fence_proxy_async();
        __syncthreads();
        if (issuer && valid) {
            if (remote) {
                // the slots we overwrite are the peer's source for its twin tile: wait until
                // the twin's loads have landed (it flags the same iteration)
                if (lane == 0) {
                    unsigned long long seen;
                    do {
                        asm volatile("ld.acquire.sys.global.u64 %0, [%1];"
                                     : "=l"(seen)
                                     : "l"(geom.flag_mine + blockIdx.x)
                                     : "memory");
                    } while (seen < flag_val);
                }
                __syncwarp();
            }
            if (tens) {
                if (lane == 0)
                    for (int e = 0; e < (1 << geom.tm_nx); ++e) {
                        uint64_t bb = base;
                        for (int i = 0; i < geom.tm_nx; ++i)
                            bb |= static_cast<uint64_t>((e >> i) & 1) << geom.tm_x[i];
                        int32_t c[5];
                        tm_coords(bb, c);
                        tensor_store(geom.tm_rank, tmap, c, tile + static_cast<uint32_t>(e) * geom.tm_box_amps);
                    }
            } else {
                for (int k = lane; k < my_runs; k += 32) {
                    const int j = warp + NW * k;
                    const uint64_t idx = base + hi_off[j << m];
                    double2* dst = psi + idx;
                    if (fused && geom.spush && (idx & svm) != sgm)
                        dst = const_cast<double2*>(geom.peer) + (idx ^ svm);  // push: into the peer's slot
                    bulk_store(dst, tile + (j << RL), run_bytes);
                }
            }
            bulk_commit();
        }
    }
    if (issuer)
        bulk_wait_all();
}


// ---------------------------------------------------------------- JIT helpers
// Constant-foldable deposit: insert a zero at every set bit of F (ascending).
__host__ __device__ constexpr uint32_t cdeposit(uint32_t g, uint32_t F) {
    for (int p = 0; p < 32; ++p)
        if ((F >> p) & 1u) {
            const uint32_t lo = g & ((1u << p) - 1u);
            g = ((g ^ lo) << 1) | lo;
        }
    return g;
}

__host__ __device__ constexpr int cpopc(uint32_t x) {
    int c = 0;
    for (; x; x &= x - 1)
        ++c;
    return c;
}

template <int NV, int C, int T>  // CX without member rotation: pure register renaming
__device__ __forceinline__ void rb_cx_plain(double2 (&v)[NV]) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        if (!((j >> C) & 1) || ((j >> T) & 1))
            continue;
        const double2 t = v[j];
        v[j] = v[j | (1 << T)];
        v[j | (1 << T)] = t;
    }
}

// ------------------------------------------------ split register blocks (JIT)
// A 16-member register group held by a lane pair (lane, lane ^ 16): the lane with
// h = lane >> 4 holds the 8 members whose bit on the split slot S equals h, at local
// index = member index with bit S removed.  Twice the threads per group means twice
// the warps per SM for the same registers per group (latency hiding for DFMA-heavy
// passes).  Primitives not crossing the split run on the 8 local registers; before one
// that does, the pair re-splits on another slot through four 16-B shuffles.
__host__ __device__ constexpr int rb_compress(int j, int S) {  // drop bit S of a 4-bit index
    return (j & ((1 << S) - 1)) | ((j >> (S + 1)) << S);
}
__host__ __device__ constexpr int rb_expand(int x, int S, int bit) {  // insert `bit` at S
    return (x & ((1 << S) - 1)) | (bit << S) | ((x >> S) << (S + 1));
}
// the 4-bit member index with bit SO = so, bit SN = sn and the other two slots = q
__host__ __device__ constexpr int rb_member(int SO, int SN, int so, int sn, int q) {
    int j = 0, k = 0;
    for (int b = 0; b < 4; ++b) {
        if (b == SO)
            j |= so << b;
        else if (b == SN)
            j |= sn << b;
        else
            j |= ((q >> k++) & 1) << b;
    }
    return j;
}

__device__ __forceinline__ double2 shfl_xor16(double2 a) {
    double2 r;
    r.x = __shfl_xor_sync(0xffffffffu, a.x, 16);
    r.y = __shfl_xor_sync(0xffffffffu, a.y, 16);
    return r;
}

template <int SO, int SN>
__device__ __forceinline__ void rb_resplit(double2 (&v)[8], uint32_t h) {
    double2 nv[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int x0 = rb_compress(rb_member(SO, SN, 0, 0, q), SO);  // s_new = 0 (s_old = h)
        const int x1 = rb_compress(rb_member(SO, SN, 0, 1, q), SO);  // s_new = 1
        const double2 keep = h ? v[x1] : v[x0];
        const double2 send = h ? v[x0] : v[x1];
        const double2 recv = shfl_xor16(send);
        const int y0 = rb_compress(rb_member(SO, SN, 0, 0, q), SN);  // s_old = 0
        const int y1 = rb_compress(rb_member(SO, SN, 1, 0, q), SN);  // s_old = 1
        nv[y0] = h ? recv : keep;
        nv[y1] = h ? keep : recv;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
        v[i] = nv[i];
}

template <int T>  // swap the register pairs differing in local bit T (CX whose control is the split slot)
__device__ __forceinline__ void rb_flip(double2 (&v)[8]) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        if ((j >> T) & 1)
            continue;
        const double2 t = v[j];
        v[j] = v[j | (1 << T)];
        v[j | (1 << T)] = t;
    }
}

template <int S>  // 16-entry diagonal over the full member index (split on S)
__device__ __forceinline__ void rb_diag_split(double2 (&v)[8], const double2* D, uint32_t r, uint32_t h) {
#pragma unroll
    for (int x = 0; x < 8; ++x)
        v[x] = cmul(D[static_cast<uint32_t>(rb_expand(x, S, 0)) ^ (h << S) ^ r], v[x]);
}

template <int K, int NT, uint32_t F, uint32_t TCTRL, uint32_t M0, uint32_t M1, uint32_t M2, uint32_t M3,
          uint32_t ROT, int S0, int S1, typename Body, typename Epi>
__device__ __forceinline__ void jit_rblock_split(double2* tile, Body&& body, Epi&& epi) {
    static_assert((1 << (K - cpopc(F))) * 2 == NT, "split blocks need exactly two threads per group");
    constexpr uint32_t M[4] = {M0, M1, M2, M3};
    const uint32_t lane = QSV_LTID & 31u;
    const uint32_t h = lane >> 4;
    const uint32_t g = ((QSV_LTID >> 5) << 4) | (lane & 15u);
    const uint32_t r = ROT ? ((ROT >> (4 * (lane & 7))) & 15u) : 0u;
    const uint32_t offr = ((r & 1u) ? M0 : 0u) | ((r & 2u) ? M1 : 0u) | ((r & 4u) ? M2 : 0u) | ((r & 8u) ? M3 : 0u);
    const uint32_t base = cdeposit(g, F) | TCTRL | offr;
    double2 v[8];
    {
        const uint32_t b0 = base ^ (h ? M[S0] : 0u);
#pragma unroll
        for (int x = 0; x < 8; ++x) {
            const int j = rb_expand(x, S0, 0);
            v[x] = tile[b0 ^ (((j & 1) ? M0 : 0u) | ((j & 2) ? M1 : 0u) | ((j & 4) ? M2 : 0u) | ((j & 8) ? M3 : 0u))];
        }
    }
    body(v, r, h);
    const uint32_t b1 = base ^ (h ? M[S1] : 0u);
#pragma unroll
    for (int x = 0; x < 8; ++x) {
        const int j = rb_expand(x, S1, 0);
        const uint32_t idx = b1 ^ (((j & 1) ? M0 : 0u) | ((j & 2) ? M1 : 0u) | ((j & 4) ? M2 : 0u) | ((j & 8) ? M3 : 0u));
        epi(v[x], idx);
        tile[idx] = v[x];
    }
}

// Register block with every structural quantity a compile-time constant; the
// generated `body(v, r)` is the block's primitive sequence as straight-line code.
struct NoEpi {
    __device__ __forceinline__ void operator()(double2&, uint32_t) const {}
};

// Block epilogue: `epib(v, base)` sees every register of the group at once (the JIT
// emits straight-line code with the diagonal-table loads that several members share
// issued once); runs before any store.
struct NoEpiB {
    template <int NV>
    __device__ __forceinline__ void operator()(double2 (&)[NV], uint32_t) const {}
};

// `epi(v, idx)` (JIT diagonal epilogue) runs on every amplitude before it is
// written back; only used when the block covers the whole tile (TCTRL == 0).
struct IdMap {
    __device__ __forceinline__ uint32_t operator()(uint32_t x) const { return x; }
};

// PERM: the pass relabel folded into this (last, single-step, whole-tile) block: after
// every thread has computed its group, members are stored through the XOR-linear tile-bit
// permutation `map` instead of a separate relabel sweep.
template <int K, int NT, int KB, uint32_t F, uint32_t TCTRL, uint32_t M0, uint32_t M1, uint32_t M2, uint32_t M3,
          uint32_t ROT, bool PERM = false, typename Body, typename Epi = NoEpi, typename EpiB = NoEpiB,
          typename Map = IdMap>
__device__ __forceinline__ void jit_rblock(double2* tile, Body&& body, Epi&& epi = Epi{}, EpiB&& epib = EpiB{},
                                           Map&& map = Map{}) {
    constexpr int NV = 1 << KB;
    constexpr uint32_t groups = 1u << (K - cpopc(F));
    constexpr uint32_t dstep = cdeposit(NT, F);
    constexpr uint32_t steps = groups >= static_cast<uint32_t>(NT) ? groups / NT : 1u;
    if (groups < static_cast<uint32_t>(NT) && QSV_LTID >= groups)
        return;
    const uint32_t r0 = ROT ? ((ROT >> (4 * (QSV_LTID & 7))) & 15u) : 0u;
    auto rot_off = [](uint32_t rr) {
        return ((rr & 1u) ? M0 : 0u) | ((rr & 2u) ? M1 : 0u) | ((rr & 4u) ? M2 : 0u) | ((rr & 8u) ? M3 : 0u);
    };
    const uint32_t offr = rot_off(r0);
    uint32_t b = cdeposit(QSV_LTID, F);
#pragma unroll 1
    for (uint32_t st = 0; st < steps; ++st) {
        const uint32_t base_in = b | TCTRL | offr;
        double2 v[NV];
#pragma unroll
        for (int j = 0; j < NV; ++j)
            v[j] = tile[base_in ^ (((j & 1) ? M0 : 0u) | ((j & 2) ? M1 : 0u) | ((j & 4) ? M2 : 0u) | ((j & 8) ? M3 : 0u))];
        uint32_t r = r0;
        body(v, r);  // may update the rotation (CX on a rotated control)
        const uint32_t base = b | TCTRL | rot_off(r);
        epib(v, base);
        if constexpr (PERM) {
            static_assert(groups == static_cast<uint32_t>(NT), "folded relabel needs one group per thread");
            __syncthreads();  // every member has been read before any permuted store
            const uint32_t mb = map(base);
#pragma unroll
            for (int j = 0; j < NV; ++j) {
                const uint32_t off = ((j & 1) ? M0 : 0u) | ((j & 2) ? M1 : 0u) | ((j & 4) ? M2 : 0u) | ((j & 8) ? M3 : 0u);
                epi(v[j], base ^ off);
                tile[mb ^ map(off)] = v[j];
            }
        } else {
#pragma unroll
            for (int j = 0; j < NV; ++j) {
                const uint32_t idx = base ^ (((j & 1) ? M0 : 0u) | ((j & 2) ? M1 : 0u) | ((j & 4) ? M2 : 0u) | ((j & 8) ? M3 : 0u));
                epi(v[j], idx);
                tile[idx] = v[j];
            }
        }
        b = ((b | F) + dstep) & ~F;
    }
}

// Structure-class form of jit_rblock (JIT class mode, programs with many distinct passes):
// the enumeration masks, member slots and rotation table are read from the op record at
// run time, so passes that differ only in qubit positions share one kernel.  `epib(v,
// base, m0, m1, m2, m3)` sees the member masks; with PERM the pass relabel `rl` (a
// RELABEL op record: destination of tile bit b in tpos[b] / xbit[b - 8]) is folded into
// the stores.
__device__ __forceinline__ uint32_t relabel_map(const TileOp& rl, int K, uint32_t x) {
    uint32_t y = 0;
    for (int b = 0; b < K; ++b)
        y |= ((x >> b) & 1u) << (b < 8 ? rl.tpos[b] : rl.xbit[b - 8]);
    return y;
}

template <int K, int NT, int KB, bool PERM = false, typename Body, typename EpiB>
__device__ __forceinline__ void jit_rblock_rt(double2* tile, const TileOp& op, Body&& body, EpiB&& epib,
                                              const TileOp* rl = nullptr) {
    constexpr int NV = 1 << KB;
    const int nfix = op.nfix;
    const uint32_t F = op.fmask, tctrl = op.tctrl;
    const uint32_t groups = 1u << (K - nfix);
    if (groups < static_cast<uint32_t>(NT) && QSV_LTID >= groups)
        return;
    const uint32_t steps = groups >= static_cast<uint32_t>(NT) ? groups / NT : 1u;
    const uint32_t dstep = deposit(NT, op.fixpos, nfix);
    const uint32_t m0 = 1u << op.tpos[0], m1 = 1u << op.tpos[1], m2 = 1u << op.tpos[2],
                   m3 = KB > 3 ? 1u << op.tpos[3] : 0u;
    auto moff = [&](uint32_t j) {
        return ((j & 1u) ? m0 : 0u) | ((j & 2u) ? m1 : 0u) | ((j & 4u) ? m2 : 0u) | ((j & 8u) ? m3 : 0u);
    };
    const uint32_t r0 = (op.rot_tab >> (4 * (QSV_LTID & 7))) & 15u;
    const uint32_t offr = moff(r0);
    uint32_t b = deposit(QSV_LTID, op.fixpos, nfix);
#pragma unroll 1
    for (uint32_t st = 0; st < steps; ++st) {
        const uint32_t base_in = b | tctrl | offr;
        double2 v[NV];
#pragma unroll
        for (int j = 0; j < NV; ++j)
            v[j] = tile[base_in ^ moff(static_cast<uint32_t>(j))];
        uint32_t r = r0;
        body(v, r);
        const uint32_t base = b | tctrl | moff(r);
        epib(v, base, m0, m1, m2, m3);
        if constexpr (PERM) {
            __syncthreads();  // every member has been read before any permuted store
            const uint32_t mb = relabel_map(*rl, K, base);
            const uint32_t q0 = relabel_map(*rl, K, m0), q1 = relabel_map(*rl, K, m1),
                           q2 = relabel_map(*rl, K, m2), q3 = relabel_map(*rl, K, m3);
#pragma unroll
            for (int j = 0; j < NV; ++j)
                tile[mb ^ (((j & 1) ? q0 : 0u) | ((j & 2) ? q1 : 0u) | ((j & 4) ? q2 : 0u) | ((j & 8) ? q3 : 0u))] = v[j];
        } else {
#pragma unroll
            for (int j = 0; j < NV; ++j)
                tile[base ^ moff(static_cast<uint32_t>(j))] = v[j];
        }
        b = next_group(b, F, dstep);
    }
}

} // namespace qsv
