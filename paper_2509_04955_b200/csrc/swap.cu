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

int fail_cuda(const char* what, cudaError_t e) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return QSV_E_CUDA;
}

int fail_nccl(const char* what, ncclResult_t r) {
    set_error(std::string(what) + ": " + ncclGetErrorString(r));
    return QSV_E_NCCL;
}

} // namespace

void join_swap(qsv_ctx* ctx) {
    cudaEventRecord(ctx->ev_a, ctx->comm_stream);
    cudaEventRecord(ctx->ev_b, ctx->copy_stream);
    cudaStreamWaitEvent(ctx->stream, ctx->ev_a, 0);
    cudaStreamWaitEvent(ctx->stream, ctx->ev_b, 0);
}

int run_swap(qsv_state* st, int g, int v, int chunk_log2, int nbuf, std::vector<cudaEvent_t>* chunk_done) {
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
    const uint64_t C = 1ull << chunk_log2;
    const uint64_t nchunks = (1ull << (l - 1)) / C;
    const bool contiguous = v >= chunk_log2;
    const size_t need = static_cast<size_t>(nbuf) * C * sizeof(double2) * (contiguous ? 1 : 2);
    if (ctx->stage_bytes < need) {
        cudaStreamSynchronize(ctx->comm_stream);
        cudaStreamSynchronize(ctx->copy_stream);
        if (ctx->d_stage)
            cudaFree(ctx->d_stage);
        ctx->d_stage = nullptr;
        ctx->stage_bytes = 0;
        e = cudaMalloc(&ctx->d_stage, need);
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
        if (r != ncclSuccess || r2 != ncclSuccess) {
            rc = fail_nccl("qsv_swap: ncclSend/ncclRecv", r != ncclSuccess ? r : r2);
            break;
        }
        cudaEventRecord(recv_ev[b], ctx->comm_stream);
        cudaStreamWaitEvent(ctx->copy_stream, recv_ev[b], 0);
        if (contiguous) {
            e = cudaMemcpyAsync(dst_contig, recv_stage + b * C, C * sizeof(double2), cudaMemcpyDeviceToDevice,
                                ctx->copy_stream);
            if (e != cudaSuccess)
                rc = fail_cuda("qsv_swap: copy-back", e);
        } else {
            scatter_half_kernel<<<grid, tb, 0, ctx->copy_stream>>>(st->amps, recv_stage + b * C, r0, C, v,
                                                                  sendbit);
        }
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
