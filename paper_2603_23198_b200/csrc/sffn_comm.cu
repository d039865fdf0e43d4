// sffn_comm.cu — hidden-dim sharding across GPUs (north_star (5)): the library's own NCCL communicator,
// one bf16 sum all-reduce of the partial outputs per FFN, optionally chunked over M so the all-reduce
// of chunk i runs on an internal communication stream while chunk i+1 computes (event-ordered).
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstring>
#include <vector>

#include "../../include/sffn.h"

struct sffn_comm {
    ncclComm_t nccl = nullptr;
    int nranks = 0, rank = 0, device = 0;
    cudaStream_t comm_stream = nullptr;
    std::vector<cudaEvent_t> events;  // per-chunk "compute done" events (+1 "comm done")
};

static int ensure_events(sffn_comm* c, int n) {
    while (static_cast<int>(c->events.size()) < n + 1) {
        cudaEvent_t e;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return SFFN_ERR_CUDA;
        c->events.push_back(e);
    }
    return SFFN_OK;
}

extern "C" {

int sffn_comm_unique_id(void* id128) {
    if (!id128) return SFFN_ERR_INVALID_ARG;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return SFFN_ERR_NCCL;
    std::memcpy(id128, &id, sizeof(id));
    return SFFN_OK;
}

int sffn_comm_init(sffn_comm** out, int nranks, int rank, const void* id128, int cuda_device) {
    if (!out || !id128 || nranks < 1 || rank < 0 || rank >= nranks) return SFFN_ERR_INVALID_ARG;
    *out = nullptr;
    if (cudaSetDevice(cuda_device) != cudaSuccess) return SFFN_ERR_CUDA;
    sffn_comm* c = new sffn_comm();
    c->nranks = nranks;
    c->rank = rank;
    c->device = cuda_device;
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    if (ncclCommInitRank(&c->nccl, nranks, id, rank) != ncclSuccess) {
        delete c;
        return SFFN_ERR_NCCL;
    }
    if (cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking) != cudaSuccess) {
        ncclCommDestroy(c->nccl);
        delete c;
        return SFFN_ERR_CUDA;
    }
    *out = c;
    return SFFN_OK;
}

int sffn_comm_destroy(sffn_comm* c) {
    if (!c) return SFFN_ERR_INVALID_ARG;
    int r = SFFN_OK;
    if (c->comm_stream) cudaStreamSynchronize(c->comm_stream);
    for (cudaEvent_t e : c->events) cudaEventDestroy(e);
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    if (c->nccl && ncclCommDestroy(c->nccl) != ncclSuccess) r = SFFN_ERR_NCCL;
    delete c;
    return r;
}

int sffn_comm_size(const sffn_comm* c) { return c ? c->nranks : -1; }

int sffn_allreduce_bf16(sffn_comm* c, void* buf, int64_t count, void* stream) {
    if (!c || !buf || count < 0) return SFFN_ERR_INVALID_ARG;
    if (count == 0) return SFFN_OK;
    if (ncclAllReduce(buf, buf, static_cast<size_t>(count), ncclBfloat16, ncclSum, c->nccl,
                      reinterpret_cast<cudaStream_t>(stream)) != ncclSuccess)
        return SFFN_ERR_NCCL;
    return SFFN_OK;
}

int sffn_sharded_forward(sffn_comm* c, const void* X, const void* Wg_s, const void* Wu_s, const void* Wd_s, int64_t M,
                         int64_t K, int64_t N_local, int T, int C, void* Y, void* workspace, size_t ws_bytes,
                         uint32_t* d_overflow, int algo, int n_chunks, void* stream) {
    if (!c) return SFFN_ERR_INVALID_ARG;
    if (n_chunks < 1) n_chunks = 1;
    if (M < 0) return SFFN_ERR_SHAPE;
    if (ws_bytes < sffn_forward_workspace_bytes(M, K, N_local, T, C, algo)) return SFFN_ERR_SHAPE;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (n_chunks == 1 || M < 2 * 128) {
        int r = sffn_forward(X, Wg_s, Wu_s, Wd_s, M, K, N_local, T, C, Y, workspace, ws_bytes, d_overflow, algo,
                             stream);
        if (r != SFFN_OK) return r;
        return sffn_allreduce_bf16(c, Y, M * K, stream);
    }
    if (ensure_events(c, n_chunks) != SFFN_OK) return SFFN_ERR_CUDA;
    // chunk rows rounded to the GEMM row tile (128) so every chunk but the last is full
    int64_t rows = (M + n_chunks - 1) / n_chunks;
    rows = (rows + 127) / 128 * 128;
    const char* x = static_cast<const char*>(X);
    char* y = static_cast<char*>(Y);
    // the comm stream must not start before earlier work on `stream` that touched Y
    if (cudaEventRecord(c->events[n_chunks], st) != cudaSuccess) return SFFN_ERR_CUDA;
    if (cudaStreamWaitEvent(c->comm_stream, c->events[n_chunks], 0) != cudaSuccess) return SFFN_ERR_CUDA;
    int i = 0;
    for (int64_t r0 = 0; r0 < M; r0 += rows, ++i) {
        const int64_t mr = (M - r0) < rows ? (M - r0) : rows;
        const size_t xoff = static_cast<size_t>(r0 * K) * 2;
        // the workspace is reused by every chunk: chunk i+1's compute follows chunk i's on `stream`
        int r = sffn_forward(x + xoff, Wg_s, Wu_s, Wd_s, mr, K, N_local, T, C, y + xoff, workspace, ws_bytes,
                             d_overflow, algo, stream);
        if (r != SFFN_OK) return r;
        if (cudaEventRecord(c->events[i], st) != cudaSuccess) return SFFN_ERR_CUDA;
        if (cudaStreamWaitEvent(c->comm_stream, c->events[i], 0) != cudaSuccess) return SFFN_ERR_CUDA;
        if ((r = sffn_allreduce_bf16(c, y + xoff, mr * K, c->comm_stream)) != SFFN_OK) return r;
    }
    if (cudaEventRecord(c->events[n_chunks], c->comm_stream) != cudaSuccess) return SFFN_ERR_CUDA;
    if (cudaStreamWaitEvent(st, c->events[n_chunks], 0) != cudaSuccess) return SFFN_ERR_CUDA;
    return SFFN_OK;
}

}  // extern "C"
