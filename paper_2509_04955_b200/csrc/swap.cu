// BBOP qubit swap over NVLink (Table 2 :332-353).
//
// The reference exchanges amplitude halves per remote gate through MPI with
// 2^b-amplitude batches and B receive buffers, the lower rank computing.  On
// one NVSwitch box every GPU reaches every peer at full bandwidth, so the B200
// design swaps the *qubit* instead: global qubit g and local qubit v trade
// places (a relabelling tracked by the host planner), after which every gate on
// the old global qubit is local.  Rank r (bit a = r_{g-l}) owns the amplitudes
// with bit v = !a that must move; its peer r ^ 2^{g-l} (Eq. 5) owns
// the matching ones, and the received amplitudes land exactly in the vacated
// slots, so the swap is in place apart from nbuf chunk buffers:
//
//   comm stream : [gather chunk c -> send stage]  ncclSend/ncclRecv(chunk c)
//   copy stream :                                 wait(c) -> copy/scatter back
//
// With nbuf >= 2 the copy-back of chunk c overlaps the transfer of chunk c+1
// (the "With Buff" row of Table 2); per-rank memory is 2^l + nbuf*2^b
// amplitudes (+ nbuf*2^b send staging when bit v lies inside a chunk).
#include "qsv_internal.h"

#include <unistd.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

namespace qsv {

namespace {

__device__ __forceinline__ uint64_t insert_bit(uint64_t r, int v, uint64_t bit) {
    const uint64_t lo = r & ((1ull << v) - 1ull);
    return ((r ^ lo) << 1) | (bit << v) | lo;
}

__global__ void gather_half_kernel(const double2* __restrict__ psi, double2* __restrict__ stage,
                                   uint64_t r0, uint64_t count, int v, uint64_t bit) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        stage[i] = psi[insert_bit(r0 + i, v, bit)];
}

__global__ void scatter_half_kernel(double2* __restrict__ psi, const double2* __restrict__ stage,
                                    uint64_t r0, uint64_t count, int v, uint64_t bit) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        psi[insert_bit(r0 + i, v, bit)] = stage[i];
}

// NVLink P2P swap: rank a = 0 exchanges pairs r in [0, H/2), rank a = 1 the rest;
// each pair is (my slot with bit v = !a) <-> (peer slot with bit v = a), read and
// written by exactly one GPU, so no staging and no copy-back.  Each thread keeps
// four remote loads in flight to cover the NVLink round trip.
__global__ void __launch_bounds__(256) p2p_swap_kernel(double2* __restrict__ mine, double2* __restrict__ theirs,
                                                       uint64_t r0, uint64_t count, int v, uint64_t mybit,
                                                       uint64_t theirbit) {
    constexpr int U = 4;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i0 = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i0 < count; i0 += stride * U) {
        double2 a[U], b[U];
        uint64_t xm[U], xt[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = i0 + u * stride;
            if (i < count) {
                xm[u] = insert_bit(r0 + i, v, mybit);
                xt[u] = insert_bit(r0 + i, v, theirbit);
                a[u] = mine[xm[u]];
                b[u] = theirs[xt[u]];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = i0 + u * stride;
            if (i < count) {
                mine[xm[u]] = b[u];
                theirs[xt[u]] = a[u];
            }
        }
    }
}

__device__ __forceinline__ uint64_t insert_zero(uint64_t x, int p) {
    const uint64_t lo = x & ((1ull << p) - 1ull);
    return ((x ^ lo) << 1) | lo;
}

// Region form of the P2P swap: pairs whose region bits equal `rval`.  Bit positions
// pos[0..npos) (ascending: v and the region bits) are inserted as zeros into the
// pair index, then the region value and the two values of bit v are ORed in.
__global__ void __launch_bounds__(256) p2p_swap_region_kernel(double2* __restrict__ mine,
                                                              double2* __restrict__ theirs, uint64_t i_begin,
                                                              uint64_t count, int p0, int p1, int p2, int npos,
                                                              uint64_t rval, uint64_t mine_v, uint64_t theirs_v) {
    constexpr int U = 4;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i0 = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i0 < count; i0 += stride * U) {
        double2 a[U], b[U];
        uint64_t xm[U], xt[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = i0 + u * stride;
            if (i < count) {
                uint64_t x = insert_zero(i_begin + i, p0);
                if (npos > 1)
                    x = insert_zero(x, p1);
                if (npos > 2)
                    x = insert_zero(x, p2);
                x |= rval;
                xm[u] = x | mine_v;
                xt[u] = x | theirs_v;
                a[u] = mine[xm[u]];
                b[u] = theirs[xt[u]];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = i0 + u * stride;
            if (i < count) {
                mine[xm[u]] = b[u];
                theirs[xt[u]] = a[u];
            }
        }
    }
}

int fail_cuda(const char* what, cudaError_t e) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return QSV_E_CUDA;
}

int fail_nccl(const char* what, ncclResult_t r) {
    set_error(std::string(what) + ": " + ncclGetErrorString(r));
    return QSV_E_NCCL;
}

struct PeerInfo {
    cudaIpcMemHandle_t handle;
    uint64_t ptr;
    int32_t pid;
    int32_t device;
    int32_t ok;
    char pad[128 - sizeof(cudaIpcMemHandle_t) - 8 - 12];
};
static_assert(sizeof(PeerInfo) == 128, "PeerInfo is exchanged as 128 bytes");

// Collective (all ranks): maps every peer's shard into this process.  Every rank
// joins both collectives whatever its local state (a failure only lowers its `ok`
// flag, which the ncclMin all-reduce combines), so no rank is left waiting.
int exchange_peers(qsv_state* st) {
    qsv_ctx* ctx = st->ctx;
    st->peers_ready = true;
    st->peer_amps.assign(ctx->nranks, nullptr);
    st->peer_ipc.assign(ctx->nranks, 0);
    PeerInfo mine{};
    mine.ok = cudaIpcGetMemHandle(&mine.handle, st->amps) == cudaSuccess;
    cudaGetLastError();
    mine.ptr = reinterpret_cast<uint64_t>(st->amps);
    mine.pid = static_cast<int32_t>(getpid());
    mine.device = ctx->device;
    unsigned char* d_info = ctx->d_coll;  // 128 B per rank, then the flag
    int* d_flag = reinterpret_cast<int*>(d_info + sizeof(PeerInfo) * ctx->nranks);
    std::vector<PeerInfo> all(ctx->nranks);
    bool local_ok = cudaMemcpy(d_info + sizeof(PeerInfo) * ctx->rank, &mine, sizeof(PeerInfo),
                               cudaMemcpyHostToDevice) == cudaSuccess;
    cudaGetLastError();
    ncclResult_t r = ncclAllGather(d_info + sizeof(PeerInfo) * ctx->rank, d_info, sizeof(PeerInfo), ncclChar,
                                   ctx->comm, ctx->comm_stream);
    if (r != ncclSuccess) {
        abort_comm(ctx, std::string("ncclAllGather: ") + ncclGetErrorString(r));
        return check_aborted(ctx, "qsv_swap: peer handle exchange");
    }
    int rc = wait_stream(ctx, ctx->comm_stream, "qsv_swap: peer handle exchange");
    if (rc != QSV_OK)
        return rc;
    local_ok = local_ok &&
               cudaMemcpy(all.data(), d_info, sizeof(PeerInfo) * ctx->nranks, cudaMemcpyDeviceToHost) == cudaSuccess;
    cudaGetLastError();
    for (int q = 0; q < ctx->nranks && local_ok; ++q) {
        if (q == ctx->rank)
            continue;
        const PeerInfo& pi = all[q];
        if (pi.pid == mine.pid) {
            int can = 0;
            cudaDeviceCanAccessPeer(&can, ctx->device, pi.device);
            if (!can)
                continue;
            const cudaError_t e = cudaDeviceEnablePeerAccess(pi.device, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
                cudaGetLastError();
                continue;
            }
            cudaGetLastError();
            st->peer_amps[q] = reinterpret_cast<double2*>(pi.ptr);
        } else if (pi.ok) {
            void* p = nullptr;
            if (cudaIpcOpenMemHandle(&p, pi.handle, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess) {
                st->peer_amps[q] = static_cast<double2*>(p);
                st->peer_ipc[q] = 1;
            } else {
                cudaGetLastError();
            }
        }
    }
    // all ranks must take the same path: P2P only if every rank mapped every peer
    int ok_local = local_ok ? 1 : 0;
    for (int q = 0; q < ctx->nranks; ++q)
        ok_local &= (q == ctx->rank || st->peer_amps[q] != nullptr) ? 1 : 0;
    int ok_all = 0;
    if (cudaMemcpy(d_flag, &ok_local, sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaGetLastError();
        // the flag cannot be set: contribute 0 through a device-side memset instead
        cudaMemsetAsync(d_flag, 0, sizeof(int), ctx->comm_stream);
    }
    r = ncclAllReduce(d_flag, d_flag, 1, ncclInt32, ncclMin, ctx->comm, ctx->comm_stream);
    if (r != ncclSuccess) {
        abort_comm(ctx, std::string("ncclAllReduce: ") + ncclGetErrorString(r));
        return check_aborted(ctx, "qsv_swap: peer map agreement");
    }
    rc = wait_stream(ctx, ctx->comm_stream, "qsv_swap: peer map agreement");
    if (rc != QSV_OK)
        return rc;
    if (cudaMemcpy(&ok_all, d_flag, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) {
        cudaGetLastError();
        ok_all = 0;
    }
    if (!ok_all) {
        for (int q = 0; q < ctx->nranks; ++q)
            if (st->peer_ipc[q] && st->peer_amps[q])
                cudaIpcCloseMemHandle(st->peer_amps[q]);
        st->peer_amps.assign(ctx->nranks, nullptr);
        st->peer_ipc.assign(ctx->nranks, 0);
    }
    return QSV_OK;
}

// Pairwise barrier with `peer` on the comm stream (an 8-byte grouped send/recv).
ncclResult_t pair_barrier(qsv_ctx* ctx, int peer) {
    ncclResult_t r = ncclGroupStart();
    if (r == ncclSuccess) r = ncclSend(ctx->d_sync, 1, ncclDouble, peer, ctx->comm, ctx->comm_stream);
    if (r == ncclSuccess) r = ncclRecv(ctx->d_sync + 1, 1, ncclDouble, peer, ctx->comm, ctx->comm_stream);
    const ncclResult_t r2 = ncclGroupEnd();
    return r != ncclSuccess ? r : r2;
}

int env_int_swap(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

bool p2p_mode() {
    const char* m = std::getenv("QSV_SWAP_MODE");
    return !(m && std::strcmp(m, "nccl") == 0);
}

} // namespace

void join_swap(qsv_ctx* ctx) {
    cudaEventRecord(ctx->ev_a, ctx->comm_stream);
    cudaEventRecord(ctx->ev_b, ctx->copy_stream);
    cudaStreamWaitEvent(ctx->stream, ctx->ev_a, 0);
    cudaStreamWaitEvent(ctx->stream, ctx->ev_b, 0);
}

bool p2p_swap_ready(qsv_state* st, int g) {
    qsv_ctx* ctx = st->ctx;
    if (!p2p_mode() || ctx->nranks < 2 || ctx->comm == nullptr)
        return false;
    if (!st->peers_ready && exchange_peers(st) != QSV_OK)  // collective: every rank reaches the same swap
        return false;
    const int l = st->n_local;
    const int peer = ctx->rank ^ (1 << (g - l));
    return st->peer_amps.size() == static_cast<size_t>(ctx->nranks) && peer < ctx->nranks && st->peer_amps[peer];
}

// Several consecutive qubit swaps (g_i <-> v_i, distinct g and distinct v) as one
// all-to-all over NVLink P2P: the 2^k ranks that differ only in the g bits
// exchange blocks pairwise — rank r's block with v bits = y goes to the rank whose g bits
// are y, which sends back its block with v bits = r's g bits — so each GPU moves
// (2^k - 1) / 2^k of its shard once instead of k / 2 of it k times.  Each pair block is
// swapped in place by the region kernel, the lower rank taking the first half of the
// pairs; grouped NCCL token send/recv with every partner bracket the exchange.
int run_multi_swap(qsv_state* st, const int* gs, const int* vs, int k) {
    qsv_ctx* ctx = st->ctx;
    const int l = st->n_local;
    if (int rc = check_aborted(ctx, "qsv_swap (multi)"); rc != QSV_OK)
        return rc;
    if (k < 2 || k > 3 || !p2p_mode() || ctx->nranks < (1 << k) || ctx->comm == nullptr)
        return QSV_E_STATE;
    if (!st->peers_ready) {
        const int rc = exchange_peers(st);
        if (rc != QSV_OK)
            return rc;
    }
    uint32_t mybits = 0;
    uint64_t gmask = 0;
    for (int i = 0; i < k; ++i) {
        mybits |= static_cast<uint32_t>((ctx->rank >> (gs[i] - l)) & 1) << i;
        gmask |= 1ull << (gs[i] - l);
    }
    // partner order: step s pairs every rank with the one whose g bits differ by s, a
    // perfect matching per step (ascending y made three ranks hit rank 0 at once)
    std::vector<int> partners;
    for (uint32_t sx = 1; sx < (1u << k); ++sx) {
        const uint32_t y = mybits ^ sx;
        int r = ctx->rank & ~static_cast<int>(gmask);
        for (int i = 0; i < k; ++i)
            r |= static_cast<int>((y >> i) & 1u) << (gs[i] - l);
        if (st->peer_amps.size() != static_cast<size_t>(ctx->nranks) || !st->peer_amps[r])
            return QSV_E_STATE;
        partners.push_back(r);
    }
    auto group_barrier = [&]() {
        ncclResult_t r = ncclGroupStart();
        for (int q : partners) {
            if (r == ncclSuccess) r = ncclSend(ctx->d_sync, 1, ncclDouble, q, ctx->comm, ctx->comm_stream);
            if (r == ncclSuccess) r = ncclRecv(ctx->d_sync + 1, 1, ncclDouble, q, ctx->comm, ctx->comm_stream);
        }
        const ncclResult_t r2 = ncclGroupEnd();
        return r != ncclSuccess ? r : r2;
    };
    cudaEventRecord(ctx->ev_a, ctx->stream);
    cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_a, 0);
    int tb = trace_open(ctx, QSV_TRACE_BARRIER, -3, 1, ctx->comm_stream);
    ncclResult_t r = group_barrier();  // every partner's earlier passes are done
    trace_close(ctx, tb, ctx->comm_stream);
    if (r != ncclSuccess)
        return fail_nccl("qsv_swap (multi): barrier", r);
    int pos[3];
    for (int i = 0; i < k; ++i)
        pos[i] = vs[i];
    std::sort(pos, pos + k);
    const uint64_t pairs = 1ull << (l - k);
    for (size_t pi = 0; pi < partners.size(); ++pi) {
        const int q = partners[pi];
        uint32_t y = 0;
        for (int i = 0; i < k; ++i)
            y |= static_cast<uint32_t>((q >> (gs[i] - l)) & 1) << i;
        uint64_t mine_v = 0, theirs_v = 0;
        for (int i = 0; i < k; ++i) {
            mine_v |= static_cast<uint64_t>((y >> i) & 1u) << vs[i];
            theirs_v |= static_cast<uint64_t>((mybits >> i) & 1u) << vs[i];
        }
        const uint64_t half = pairs / 2;
        const uint64_t begin = ctx->rank < q ? 0 : half;
        const int tk = trace_open(ctx, QSV_TRACE_SWAP, -3, 1, ctx->comm_stream);
        p2p_swap_region_kernel<<<ctx->sm_count * 4, 256, 0, ctx->comm_stream>>>(
            st->amps, st->peer_amps[q], begin, half, pos[0], k > 1 ? pos[1] : 0, k > 2 ? pos[2] : 0, k, 0ull, mine_v,
            theirs_v);
        trace_close(ctx, tk, ctx->comm_stream);
    }
    tb = trace_open(ctx, QSV_TRACE_BARRIER, -3, 1, ctx->comm_stream);
    r = group_barrier();  // every partner's writes into this shard are done
    trace_close(ctx, tb, ctx->comm_stream);
    if (r != ncclSuccess)
        return fail_nccl("qsv_swap (multi): barrier", r);
    join_swap(ctx);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? QSV_OK : fail_cuda("qsv_swap (multi): kernel", e);
}

int fused_swap_finish(qsv_state* st, int g) {
    qsv_ctx* ctx = st->ctx;
    const int peer = ctx->rank ^ (1 << (g - st->n_local));
    cudaEventRecord(ctx->ev_a, ctx->stream);
    cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_a, 0);
    const int tb = trace_open(ctx, QSV_TRACE_BARRIER, -2, 1, ctx->comm_stream);
    const ncclResult_t r = pair_barrier(ctx, peer);  // the peer's pushes into this shard are done
    trace_close(ctx, tb, ctx->comm_stream);
    if (r != ncclSuccess)
        return fail_nccl("qsv_swap (push): barrier", r);
    cudaEventRecord(ctx->ev_b, ctx->comm_stream);
    cudaStreamWaitEvent(ctx->stream, ctx->ev_b, 0);
    return QSV_OK;
}

int fused_swap_prepare(qsv_state* st, int g, int v, const Step& step, FusedSwap* out) {
    qsv_ctx* ctx = st->ctx;
    const int l = st->n_local;
    if (int rc = check_aborted(ctx, "qsv_swap (fused)"); rc != QSV_OK)
        return rc;
    if (!p2p_mode() || ctx->nranks < 2 || ctx->comm == nullptr || g < l || v < 0 || v >= l)
        return QSV_E_STATE;
    // geometry: v must not sit in the pass's contiguous low run (a run has one source)
    const PassGeom& pg = step.geom;
    if (v < pg.L)
        return QSV_E_STATE;
    int sv_tile = 0, below = 0;
    for (int i = 0; i < pg.nhigh; ++i) {
        if (pg.high[i] == v)
            sv_tile = 1;
        else if (pg.high[i] < v)
            ++below;
    }
    if (!st->peers_ready) {
        const int rc = exchange_peers(st);  // collective: every rank reaches its first swap
        if (rc != QSV_OK)
            return rc;
    }
    const int peer = ctx->rank ^ (1 << (g - l));
    if (st->peer_amps.size() != static_cast<size_t>(ctx->nranks) || !st->peer_amps[peer])
        return QSV_E_STATE;  // symmetric on one box: every rank takes the plain path
    if (!ctx->d_sync) {
        const cudaError_t e = dev_alloc(ctx, reinterpret_cast<void**>(&ctx->d_sync), 2 * sizeof(double), 3);
        if (e != cudaSuccess)
            return fail_cuda("qsv_swap: sync token cudaMalloc", e);
        cudaMemset(ctx->d_sync, 0, 2 * sizeof(double));
    }
    // both shards are final before either side reads the other's
    cudaEventRecord(ctx->ev_a, ctx->stream);
    cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_a, 0);
    const int tb = trace_open(ctx, QSV_TRACE_BARRIER, -2, 1, ctx->comm_stream);
    const ncclResult_t r = pair_barrier(ctx, peer);
    trace_close(ctx, tb, ctx->comm_stream);
    if (r != ncclSuccess)
        return fail_nccl("qsv_swap (fused): barrier", r);
    cudaEventRecord(ctx->ev_b, ctx->comm_stream);
    cudaStreamWaitEvent(ctx->stream, ctx->ev_b, 0);
    out->peer = st->peer_amps[peer];
    out->flag_mine = reinterpret_cast<unsigned long long*>(st->amps + st->size);
    out->flag_peer = reinterpret_cast<unsigned long long*>(st->peer_amps[peer] + st->size);
    out->epoch = ++st->fused_epoch;
    out->sv = v;
    out->sv_tile = sv_tile;
    out->sv_tidx = v - pg.L - below;  // v's position among the tile-index (non-tile) bits
    out->sgbit = static_cast<uint32_t>((ctx->rank >> (g - l)) & 1);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? QSV_OK : fail_cuda("qsv_swap (fused)", e);
}

int run_swap(qsv_state* st, int g, int v, int chunk_log2, int nbuf, std::vector<cudaEvent_t>* chunk_done,
             uint64_t region_mask, const std::vector<cudaEvent_t>* pre_ready) {
    qsv_ctx* ctx = st->ctx;
    const int l = st->n_local;
    int m = 0;
    while ((1 << m) < ctx->nranks)
        ++m;
    if (ctx->nranks < 2 || ctx->comm == nullptr) {
        set_error("qsv_swap: needs a multi-rank context");
        return QSV_E_STATE;
    }
    if (g < l || g >= l + m || v < 0 || v >= l || chunk_log2 < 0 || chunk_log2 > l - 1 || nbuf < 1 ||
        nbuf > 8) {
        set_error("qsv_swap: need n_local <= g < n_total, 0 <= v < n_local, chunk_log2 < n_local, 1 <= nbuf <= 8");
        return QSV_E_ARG;
    }
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e != cudaSuccess)
        return fail_cuda("cudaSetDevice", e);
    const int peer = ctx->rank ^ (1 << (g - l));
    const uint64_t a = static_cast<uint64_t>((ctx->rank >> (g - l)) & 1);
    const uint64_t sendbit = a ^ 1ull;

    if (int rc = check_aborted(ctx, "qsv_swap"); rc != QSV_OK)
        return rc;
    if (p2p_mode()) {
        if (!st->peers_ready) {
            const int rc = exchange_peers(st);  // collective: every rank reaches its first swap
            if (rc != QSV_OK)
                return rc;
        }
        // every rank must agree on the mode: P2P only when both sides mapped each other,
        // which holds symmetrically on one NVSwitch box (checked per pair below)
    }
    if (p2p_mode() && st->peer_amps.size() == static_cast<size_t>(ctx->nranks) && st->peer_amps[peer]) {
        if (!ctx->d_sync) {
            e = dev_alloc(ctx, reinterpret_cast<void**>(&ctx->d_sync), 2 * sizeof(double), 3);
            if (e != cudaSuccess)
                return fail_cuda("qsv_swap: sync token cudaMalloc", e);
            cudaMemset(ctx->d_sync, 0, 2 * sizeof(double));
        }
        region_mask &= ~(1ull << v);
        const bool fed = pre_ready && chunk_done && region_mask != 0 && pre_ready->size() == 4;
        ncclResult_t r = ncclSuccess;
        if (!fed) {
            cudaEventRecord(ctx->ev_a, ctx->stream);
            cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_a, 0);
            const int tb0 = trace_open(ctx, QSV_TRACE_BARRIER, -1, 1, ctx->comm_stream);
            r = pair_barrier(ctx, peer);  // the peer's earlier passes are done
            trace_close(ctx, tb0, ctx->comm_stream);
            if (r != ncclSuccess)
                return fail_nccl("qsv_swap: barrier", r);
        }
        const uint64_t H = 1ull << (l - 1);
        const uint64_t half = H / 2;
        if (!chunk_done || region_mask == 0) {
            const int tk = trace_open(ctx, QSV_TRACE_SWAP, -1, 1, ctx->comm_stream);
            p2p_swap_kernel<<<ctx->sm_count * 4, 256, 0, ctx->comm_stream>>>(st->amps, st->peer_amps[peer],
                                                                             a * half, half, v, sendbit, a);
            trace_close(ctx, tk, ctx->comm_stream);
            const int tb1 = trace_open(ctx, QSV_TRACE_BARRIER, -1, 1, ctx->comm_stream);
            r = pair_barrier(ctx, peer);  // the peer's writes into this shard are done
            trace_close(ctx, tb1, ctx->comm_stream);
            if (r != ncclSuccess)
                return fail_nccl("qsv_swap: barrier", r);
            if (chunk_done) {
                cudaEvent_t ev;
                cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
                cudaEventRecord(ev, ctx->comm_stream);
                chunk_done->push_back(ev);
            } else {
                join_swap(ctx);
            }
        } else {
            // one kernel + pair barrier per region: region c is final when its event fires
            int pos[3], npos = 0, rb[2], nr = 0;
            for (int b = 0; b < l && npos < 3; ++b)
                if (b == v || ((region_mask >> b) & 1ull)) {
                    pos[npos++] = b;
                    if (b != v)
                        rb[nr++] = b;
                }
            const uint64_t pairs = H >> nr;  // per region, both ranks together
            const uint64_t mine_half = pairs / 2;
            const int sms = std::max(1, std::min(ctx->sm_count, env_int_swap("QSV_SWAP_SMS", 16)));
            for (uint64_t c = 0; c < (1ull << nr); ++c) {
                if (fed) {
                    // region c of the passes before the swap is written on both sides
                    cudaStreamWaitEvent(ctx->comm_stream, (*pre_ready)[c], 0);
                    r = pair_barrier(ctx, peer);
                    if (r != ncclSuccess)
                        return fail_nccl("qsv_swap: barrier", r);
                }
                uint64_t rval = 0;
                for (int i = 0; i < nr; ++i)
                    rval |= ((c >> i) & 1ull) << rb[i];
                const int tk = trace_open(ctx, QSV_TRACE_SWAP, static_cast<int>(c), 1, ctx->comm_stream);
                p2p_swap_region_kernel<<<sms * 4, 256, 0, ctx->comm_stream>>>(
                    st->amps, st->peer_amps[peer], a * mine_half, mine_half, pos[0], npos > 1 ? pos[1] : 0,
                    npos > 2 ? pos[2] : 0, npos, rval, sendbit << v, a << v);
                trace_close(ctx, tk, ctx->comm_stream);
                r = pair_barrier(ctx, peer);
                if (r != ncclSuccess)
                    return fail_nccl("qsv_swap: barrier", r);
                cudaEvent_t ev;
                cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
                cudaEventRecord(ev, ctx->comm_stream);
                chunk_done->push_back(ev);
            }
        }
        e = cudaGetLastError();
        return e == cudaSuccess ? QSV_OK : fail_cuda("qsv_swap: p2p kernel", e);
    }
    const uint64_t C = 1ull << chunk_log2;
    const uint64_t nchunks = (1ull << (l - 1)) / C;
    const bool contiguous = v >= chunk_log2;
    const size_t need = static_cast<size_t>(nbuf) * C * sizeof(double2) * (contiguous ? 1 : 2);
    if (ctx->stage_bytes < need) {
        if (int rc = wait_stream(ctx, ctx->comm_stream, "qsv_swap: staging resize"); rc != QSV_OK)
            return rc;
        if (int rc = wait_stream(ctx, ctx->copy_stream, "qsv_swap: staging resize"); rc != QSV_OK)
            return rc;
        if (ctx->d_stage)
            dev_free(ctx, ctx->d_stage, 1);
        ctx->d_stage = nullptr;
        ctx->stage_bytes = 0;
        e = dev_alloc(ctx, &ctx->d_stage, need, 1);
        if (e != cudaSuccess)
            return fail_cuda("qsv_swap: staging cudaMalloc", e);
        ctx->stage_bytes = need;
    }
    double2* recv_stage = static_cast<double2*>(ctx->d_stage);
    double2* send_stage = recv_stage + static_cast<size_t>(nbuf) * C;

    std::vector<cudaEvent_t> recv_ev(nbuf), free_ev(nbuf);
    for (int b = 0; b < nbuf; ++b) {
        cudaEventCreateWithFlags(&recv_ev[b], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&free_ev[b], cudaEventDisableTiming);
    }
    // fork: both helper streams start after all work queued so far
    cudaEventRecord(ctx->ev_a, ctx->stream);
    cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_a, 0);
    cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_a, 0);
    const int tb = 256;
    const int grid = ctx->sm_count * 4;
    int rc = QSV_OK;
    for (uint64_t c = 0; c < nchunks && rc == QSV_OK; ++c) {
        const int b = static_cast<int>(c % nbuf);
        if (c >= static_cast<uint64_t>(nbuf))
            cudaStreamWaitEvent(ctx->comm_stream, free_ev[b], 0);  // stage b copied back
        const uint64_t r0 = c * C;
        const double2* src;
        double2* dst_contig = nullptr;
        // the send/recv record covers the send-side gather too (same stream, same chunk)
        const int ts = trace_open(ctx, QSV_TRACE_SENDRECV, static_cast<int>(c), 1, ctx->comm_stream);
        if (contiguous) {
            dst_contig = st->amps + ((r0 >> v) << (v + 1)) + (sendbit << v) + (r0 & ((1ull << v) - 1ull));
            src = dst_contig;
        } else {
            gather_half_kernel<<<grid, tb, 0, ctx->comm_stream>>>(st->amps, send_stage + b * C, r0, C, v,
                                                                 sendbit);
            src = send_stage + b * C;
        }
        ncclResult_t r = ncclGroupStart();
        if (r == ncclSuccess) r = ncclSend(src, 2 * C, ncclDouble, peer, ctx->comm, ctx->comm_stream);
        if (r == ncclSuccess) r = ncclRecv(recv_stage + b * C, 2 * C, ncclDouble, peer, ctx->comm, ctx->comm_stream);
        ncclResult_t r2 = ncclGroupEnd();
        trace_close(ctx, ts, ctx->comm_stream);
        if (r != ncclSuccess || r2 != ncclSuccess) {
            rc = fail_nccl("qsv_swap: ncclSend/ncclRecv", r != ncclSuccess ? r : r2);
            break;
        }
        cudaEventRecord(recv_ev[b], ctx->comm_stream);
        cudaStreamWaitEvent(ctx->copy_stream, recv_ev[b], 0);
        const int tc = trace_open(ctx, QSV_TRACE_COPYBACK, static_cast<int>(c), 2, ctx->copy_stream);
        if (contiguous) {
            e = cudaMemcpyAsync(dst_contig, recv_stage + b * C, C * sizeof(double2), cudaMemcpyDeviceToDevice,
                                ctx->copy_stream);
            if (e != cudaSuccess)
                rc = fail_cuda("qsv_swap: copy-back", e);
        } else {
            scatter_half_kernel<<<grid, tb, 0, ctx->copy_stream>>>(st->amps, recv_stage + b * C, r0, C, v,
                                                                  sendbit);
        }
        trace_close(ctx, tc, ctx->copy_stream);
        cudaEventRecord(free_ev[b], ctx->copy_stream);
        if (chunk_done) {
            // region c of the shard (half-index chunk c, both values of bit v) is final
            cudaEvent_t ev;
            cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
            cudaEventRecord(ev, ctx->copy_stream);
            chunk_done->push_back(ev);
        }
    }
    // join: the compute stream continues after both helper streams (deferred to
    // the caller when it overlaps region passes with the chunks)
    if (!chunk_done)
        join_swap(ctx);
    for (int b = 0; b < nbuf; ++b) {
        cudaEventDestroy(recv_ev[b]);
        cudaEventDestroy(free_ev[b]);
    }
    e = cudaGetLastError();
    if (rc == QSV_OK && e != cudaSuccess)
        rc = fail_cuda("qsv_swap", e);
    return rc;
}

} // namespace qsv
