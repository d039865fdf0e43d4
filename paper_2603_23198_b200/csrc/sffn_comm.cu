// sffn_comm.cu — hidden-dim sharding across GPUs (north_star (5)): the library's own NCCL communicator,
// one bf16 sum all-reduce of the partial outputs per FFN, optionally chunked over M so the all-reduce
// of chunk i runs on an internal communication stream while chunk i+1 computes (event-ordered).
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>  // NCCL 2.28 device API: symmetric windows, LSA peer pointers, multimem, LSA barriers

#include <cuda_bf16.h>

#include <cstring>
#include <vector>

#include "../../include/sffn.h"

struct sffn_comm {
    ncclComm_t nccl = nullptr;
    int nranks = 0, rank = 0, device = 0;
    cudaStream_t comm_stream = nullptr;
    std::vector<cudaEvent_t> events;  // per-chunk "compute done" events (+1 "comm done")
    // NEXT-3 symmetric path (sffn_comm_symmetric_init): one registered window holding this rank's partial Y
    void* sym_buf = nullptr;
    size_t sym_bytes = 0;
    int64_t sym_rows = 0, sym_K = 0;
    ncclWindow_t win = nullptr;
    ncclDevComm dev{};
    bool has_dev = false, multimem = false;
    // fused window-granular all-reduce (sffn_sharded_forward_fused).  Device table d_ptrs: [0, G) peer window
    // bases, [G] multicast base (0 if none), [G + 1] byte offset of the counter set the next call uses.  Two sets
    // of per-window arrival counters follow the partial-Y region; each call's closing kernel zeroes the set it used
    // (after the barrier: no rank can still touch it) and flips [G + 1] — device-side, so graph replays alternate.
    uint64_t* d_ptrs = nullptr;
    int64_t flags_off = 0, nwin = 0;
};

extern "C" int sffn__forward_fused(const void* X, const void* Wg, const void* Wu, const void* Wd, int64_t M, int64_t K,
                                   int64_t N, int T, int C, void* Y, void* workspace, size_t ws_bytes,
                                   uint32_t* d_overflow, const uint64_t* ptrs, int G, int rank, int phase,
                                   void* stream);

// device: ptrs[p] = rank p's window base through the LSA mapping, ptrs[G] = the window's multicast address (or 0),
// ptrs[G + 1] = the first counter set's offset
__global__ void sym_ptrs_kernel(ncclDevComm dc, ncclWindow_t win, int G, int multimem, int64_t flags_off,
                                uint64_t* ptrs) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int p = 0; p < G; ++p) ptrs[p] = reinterpret_cast<uint64_t>(ncclGetLsaPointer(win, 0, p));
    ptrs[G] = multimem ? reinterpret_cast<uint64_t>(ncclGetLsaMultimemPointer(win, 0, dc)) : 0ull;
    ptrs[G + 1] = static_cast<uint64_t>(flags_off);
}

// ---------------------------------------------------------------- NEXT-3: symmetric-memory all-reduce kernel
// One launch after the DOWN GEMM (whose epilogue wrote this rank's partial Y straight into the registered
// window).  Every rank owns 1/G of the 16-byte chunks of Y:
//   LSA barrier (all ranks' partials are in their windows)
//   multimem path (NVSwitch NVLS): multimem.ld_reduce.add.acc::f32 of the chunk through the multicast address
//     (the switch reads the G copies and returns their fp32-accumulated bf16 sum), multimem.st of the result
//     (the switch writes it into every rank's window);
//   LSA path (no multicast object): loads of the chunk from every peer's window over NVLink (P2P), fp32 sum,
//     stores of the bf16 result into every peer's window;
//   LSA barrier (every slice is back in every window), then the local copy window -> Y.
// Rank r reads and writes only its own slice in every window, so the reduction is in place without races.
constexpr int SYM_CTAS = 128;
constexpr int SYM_THREADS = 512;

__device__ __forceinline__ void bf16x8_acc(float (&a)[8], const uint4& v) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        a[2 * i] += __uint_as_float(w[i] << 16);
        a[2 * i + 1] += __uint_as_float(w[i] & 0xFFFF0000u);
    }
}
__device__ __forceinline__ uint32_t bf16x2_rn(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}

// Grid-stride loops over 16-byte elements [q0, q1) with SYM_U independent loads in flight per thread before the
// stores (one load per iteration leaves the copy latency bound at ~3 TB/s).
constexpr int SYM_U = 4;
__device__ __forceinline__ void sym_copy(const uint4* src, uint4* dst, int64_t q0, int64_t q1) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t qb = q0 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; qb < q1; qb += SYM_U * stride) {
        uint4 v[SYM_U];
#pragma unroll
        for (int u = 0; u < SYM_U; ++u)
            if (qb + u * stride < q1) v[u] = src[qb + u * stride];
#pragma unroll
        for (int u = 0; u < SYM_U; ++u)
            if (qb + u * stride < q1) dst[qb + u * stride] = v[u];
    }
}
// sum over the ranks' windows of [q0, q1): multimem.ld_reduce through the switch (mc != null), else P2P loads with
// fp32 accumulation; the result goes to every window (bcast: multimem.st / P2P stores) or to out[q - q0]
__device__ __forceinline__ void sym_reduce(ncclWindow_t win, uint4* mc, int nranks, int64_t q0, int64_t q1, bool bcast,
                                           uint4* out) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t qb = q0 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; qb < q1; qb += SYM_U * stride) {
        uint4 v[SYM_U];
        if (mc) {
#pragma unroll
            for (int u = 0; u < SYM_U; ++u)
                if (qb + u * stride < q1)
                    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                                 : "l"(mc + qb + u * stride)
                                 : "memory");
        } else {
            float a[SYM_U][8];
#pragma unroll
            for (int u = 0; u < SYM_U; ++u)
#pragma unroll
                for (int i = 0; i < 8; ++i) a[u][i] = 0.f;
            for (int p = 0; p < nranks; ++p) {
                const uint4* src = static_cast<const uint4*>(ncclGetLsaPointer(win, 0, p));
                uint4 t[SYM_U];
#pragma unroll
                for (int u = 0; u < SYM_U; ++u)
                    t[u] = qb + u * stride < q1 ? __ldcg(src + qb + u * stride) : make_uint4(0, 0, 0, 0);
#pragma unroll
                for (int u = 0; u < SYM_U; ++u) bf16x8_acc(a[u], t[u]);
            }
#pragma unroll
            for (int u = 0; u < SYM_U; ++u)
                v[u] = make_uint4(bf16x2_rn(a[u][0], a[u][1]), bf16x2_rn(a[u][2], a[u][3]),
                                  bf16x2_rn(a[u][4], a[u][5]), bf16x2_rn(a[u][6], a[u][7]));
        }
#pragma unroll
        for (int u = 0; u < SYM_U; ++u) {
            const int64_t q = qb + u * stride;
            if (q >= q1) continue;
            if (!bcast) {
                out[q - q0] = v[u];
            } else if (mc) {
                asm volatile("multimem.st.relaxed.sys.global.v4.bf16x2 [%0], {%1,%2,%3,%4};" ::"l"(mc + q),
                             "r"(v[u].x), "r"(v[u].y), "r"(v[u].z), "r"(v[u].w)
                             : "memory");
            } else {
                for (int p = 0; p < nranks; ++p) static_cast<uint4*>(ncclGetLsaPointer(win, 0, p))[q] = v[u];
            }
        }
    }
}

// Reduce-scatter variant (sequence-parallel consumers): rank r reduces its 1/G slice of rows
// [row0, row1) from every window (multimem.ld_reduce, or P2P loads) and writes it only to its own output; one LSA
// barrier before (partials complete everywhere) and one after (no rank overwrites its window, i.e. starts the next
// forward, while a peer may still be reading it).
__global__ void __launch_bounds__(SYM_THREADS) sym_reduce_scatter_kernel(ncclDevComm dc, ncclWindow_t win, int64_t q0,
                                                                        int64_t q1, int nranks, int multimem,
                                                                        uint4* Yr) {
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), blockIdx.x, multimem != 0);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
    sym_reduce(win, multimem ? static_cast<uint4*>(ncclGetLsaMultimemPointer(win, 0, dc)) : nullptr, nranks, q0, q1,
               false, Yr);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
}

// After the fused DOWN: every rank's reducers are done (LSA barrier), then the local copy window -> Y.
__global__ void __launch_bounds__(SYM_THREADS) sym_finish_kernel(ncclDevComm dc, ncclWindow_t win, int64_t n16,
                                                                int multimem, uint4* Y, uint64_t* cur_off,
                                                                int64_t flags_off, int64_t nwin_max, int64_t nwin) {
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), blockIdx.x, multimem != 0);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
    const uint4* loc = static_cast<const uint4*>(ncclGetLocalPointer(win, 0));
    if (blockIdx.x == 0) {  // this call's counter set: every rank's increments and this rank's waits are done
        const int64_t off = static_cast<int64_t>(*cur_off);
        uint32_t* flags = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(ncclGetLocalPointer(win, 0)) + off);
        for (int64_t w = threadIdx.x; w < nwin; w += blockDim.x) flags[w] = 0;
        __syncthreads();
        if (threadIdx.x == 0) *cur_off = static_cast<uint64_t>(off == flags_off ? flags_off + 4 * nwin_max : flags_off);
    }
    sym_copy(loc, Y, 0, n16);
}

__global__ void __launch_bounds__(SYM_THREADS) sym_allreduce_kernel(ncclDevComm dc, ncclWindow_t win, int64_t n16,
                                                                   int rank, int nranks, int multimem, uint4* Y) {
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), blockIdx.x, multimem != 0);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
    const int64_t q0 = n16 * rank / nranks, q1 = n16 * (rank + 1) / nranks;
    sym_reduce(win, multimem ? static_cast<uint4*>(ncclGetLsaMultimemPointer(win, 0, dc)) : nullptr, nranks, q0, q1,
               true, nullptr);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
    sym_copy(static_cast<const uint4*>(ncclGetLocalPointer(win, 0)), Y, 0, n16);
}

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
    if (c->has_dev) {
        cudaDeviceSynchronize();
        if (ncclDevCommDestroy(c->nccl, &c->dev) != ncclSuccess) r = SFFN_ERR_NCCL;
        if (c->win && ncclCommWindowDeregister(c->nccl, c->win) != ncclSuccess) r = SFFN_ERR_NCCL;
        if (c->sym_buf && ncclMemFree(c->sym_buf) != ncclSuccess) r = SFFN_ERR_NCCL;
        if (c->d_ptrs) cudaFree(c->d_ptrs);
    }
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

int sffn_comm_symmetric_init(sffn_comm* c, int64_t max_rows, int64_t K) {
    if (!c || max_rows < 1 || K < 8 || K % 8 != 0) return SFFN_ERR_INVALID_ARG;
    if (c->sym_buf) return SFFN_ERR_INVALID_ARG;  // once per communicator
    // [partial Y: max_rows x K bf16][arrival counters: one uint32 per 2048-row window]
    const int64_t flags_off = (static_cast<int64_t>(max_rows) * K * 2 + 255) / 256 * 256;
    const int64_t nwin = (max_rows + 2047) / 2048;
    const size_t bytes = (static_cast<size_t>(flags_off + 8 * nwin) + NCCL_WIN_REQUIRED_ALIGNMENT - 1) /
                         NCCL_WIN_REQUIRED_ALIGNMENT * NCCL_WIN_REQUIRED_ALIGNMENT;
    if (ncclMemAlloc(&c->sym_buf, bytes) != ncclSuccess) {
        c->sym_buf = nullptr;
        return SFFN_ERR_UNSUPPORTED;
    }
    if (ncclCommWindowRegister(c->nccl, c->sym_buf, bytes, &c->win, NCCL_WIN_COLL_SYMMETRIC) != ncclSuccess) {
        ncclMemFree(c->sym_buf);
        c->sym_buf = nullptr;
        return SFFN_ERR_UNSUPPORTED;
    }
    ncclDevCommRequirements req;
    std::memset(&req, 0, sizeof(req));
    req.lsaBarrierCount = SYM_CTAS;
    req.lsaMultimem = c->nranks > 1;  // NVLS multicast when NCCL can set it up (NVSwitch systems)
    ncclResult_t nr = ncclDevCommCreate(c->nccl, &req, &c->dev);
    if (nr != ncclSuccess && req.lsaMultimem) {  // no NVLS on this system: peer loads / stores instead
        req.lsaMultimem = false;
        nr = ncclDevCommCreate(c->nccl, &req, &c->dev);
    }
    if (nr != ncclSuccess) {
        ncclCommWindowDeregister(c->nccl, c->win);
        ncclMemFree(c->sym_buf);
        c->sym_buf = nullptr;
        c->win = nullptr;
        return SFFN_ERR_UNSUPPORTED;
    }
    // any failure from here on releases everything acquired above, so a retry starts clean
    auto release = [&](int status) {
        if (c->d_ptrs) cudaFree(c->d_ptrs);
        c->d_ptrs = nullptr;
        ncclDevCommDestroy(c->nccl, &c->dev);
        ncclCommWindowDeregister(c->nccl, c->win);
        ncclMemFree(c->sym_buf);
        c->sym_buf = nullptr;
        c->win = nullptr;
        return status;
    };
    if (cudaMemset(static_cast<uint8_t*>(c->sym_buf) + flags_off, 0, static_cast<size_t>(8 * nwin)) != cudaSuccess ||
        cudaMalloc(&c->d_ptrs, static_cast<size_t>(c->nranks + 2) * 8) != cudaSuccess)
        return release(SFFN_ERR_CUDA);
    sym_ptrs_kernel<<<1, 32>>>(c->dev, c->win, c->nranks, req.lsaMultimem ? 1 : 0, flags_off, c->d_ptrs);
    if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) return release(SFFN_ERR_CUDA);
    c->flags_off = flags_off;
    c->nwin = nwin;
    c->has_dev = true;
    c->multimem = req.lsaMultimem;
    c->sym_bytes = bytes;
    c->sym_rows = max_rows;
    c->sym_K = K;
    return SFFN_OK;
}

int sffn_comm_symmetric_info(const sffn_comm* c, int* multimem, int64_t* max_rows, int64_t* K) {
    if (!c) return SFFN_ERR_INVALID_ARG;
    if (multimem) *multimem = c->multimem ? 1 : 0;
    if (max_rows) *max_rows = c->has_dev ? c->sym_rows : 0;
    if (K) *K = c->has_dev ? c->sym_K : 0;
    return c->has_dev ? SFFN_OK : SFFN_ERR_UNSUPPORTED;
}

int sffn_allreduce_sym_bf16(sffn_comm* c, const void* src, void* Y, int64_t rows, int64_t K, void* stream) {
    if (!c || !Y || rows < 0 || K < 8 || K % 8 != 0) return SFFN_ERR_INVALID_ARG;
    if (!c->has_dev) return SFFN_ERR_UNSUPPORTED;
    if (rows > c->sym_rows || K != c->sym_K) return SFFN_ERR_SHAPE;
    if (rows == 0) return SFFN_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const size_t bytes = static_cast<size_t>(rows) * K * 2;
    if (src && src != c->sym_buf &&
        cudaMemcpyAsync(c->sym_buf, src, bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return SFFN_ERR_CUDA;
    sym_allreduce_kernel<<<SYM_CTAS, SYM_THREADS, 0, st>>>(c->dev, c->win, static_cast<int64_t>(bytes / 16), c->rank,
                                                           c->nranks, c->multimem ? 1 : 0, static_cast<uint4*>(Y));
    return cudaGetLastError() == cudaSuccess ? SFFN_OK : SFFN_ERR_CUDA;
}

int sffn_reduce_scatter_sym_bf16(sffn_comm* c, const void* src, int64_t rows, int64_t K, void* Y_slice,
                                  int64_t* row0, int64_t* nrows, void* stream) {
    if (!c || rows < 0 || K < 8 || K % 8 != 0) return SFFN_ERR_INVALID_ARG;
    if (!c->has_dev) return SFFN_ERR_UNSUPPORTED;
    if (rows > c->sym_rows || K != c->sym_K) return SFFN_ERR_SHAPE;
    // rank r owns rows [rows * r / G, rows * (r + 1) / G)
    const int64_t r0 = rows * c->rank / c->nranks, r1 = rows * (c->rank + 1) / c->nranks;
    if (row0) *row0 = r0;
    if (nrows) *nrows = r1 - r0;
    if (rows == 0) return SFFN_OK;
    if (!Y_slice && r1 > r0) return SFFN_ERR_INVALID_ARG;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (src && src != c->sym_buf &&
        cudaMemcpyAsync(c->sym_buf, src, static_cast<size_t>(rows) * K * 2, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return SFFN_ERR_CUDA;
    const int64_t k16 = K / 8;  // 16-byte chunks per row
    sym_reduce_scatter_kernel<<<SYM_CTAS, SYM_THREADS, 0, st>>>(c->dev, c->win, r0 * k16, r1 * k16, c->nranks,
                                                                c->multimem ? 1 : 0, static_cast<uint4*>(Y_slice));
    return cudaGetLastError() == cudaSuccess ? SFFN_OK : SFFN_ERR_CUDA;
}

int sffn_sharded_forward_fused(sffn_comm* c, const void* X, const void* Wg_s, const void* Wu_s, const void* Wd_s,
                               int64_t M, int64_t K, int64_t N_local, int T, int C, void* Y, void* workspace,
                               size_t ws_bytes, uint32_t* d_overflow, void* stream) {
    if (!c) return SFFN_ERR_INVALID_ARG;
    if (!c->has_dev) return SFFN_ERR_UNSUPPORTED;
    if (M < 0 || M > c->sym_rows || K != c->sym_K) return SFFN_ERR_SHAPE;
    if (!Y) return SFFN_ERR_INVALID_ARG;
    if (M == 0) return SFFN_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    // the DOWN GEMM writes the partial Y into the window and reduces each 2048-row window across the ranks as soon as
    // every rank has counted it; then one barrier (all windows reduced everywhere) and the local copy window -> Y
    int r = sffn__forward_fused(X, Wg_s, Wu_s, Wd_s, M, K, N_local, T, C, c->sym_buf, workspace, ws_bytes,
                                d_overflow, c->d_ptrs, c->nranks, c->rank, 0, stream);
    if (r != SFFN_OK) return r;
    sym_finish_kernel<<<SYM_CTAS, SYM_THREADS, 0, st>>>(c->dev, c->win, M * K / 8, c->multimem ? 1 : 0,
                                                       static_cast<uint4*>(Y), c->d_ptrs + c->nranks + 1,
                                                       c->flags_off, c->nwin, (M + 2047) / 2048);
    return cudaGetLastError() == cudaSuccess ? SFFN_OK : SFFN_ERR_CUDA;
}

int sffn_sharded_forward_sym(sffn_comm* c, const void* X, const void* Wg_s, const void* Wu_s, const void* Wd_s,
                             int64_t M, int64_t K, int64_t N_local, int T, int C, void* Y, void* workspace,
                             size_t ws_bytes, uint32_t* d_overflow, int algo, void* stream) {
    if (!c) return SFFN_ERR_INVALID_ARG;
    if (!c->has_dev) return SFFN_ERR_UNSUPPORTED;
    if (M < 0 || M > c->sym_rows || K != c->sym_K) return SFFN_ERR_SHAPE;
    if (!Y) return SFFN_ERR_INVALID_ARG;
    // the DOWN epilogue writes this rank's partial Y straight into the registered window (no staging copy)
    int r = sffn_forward(X, Wg_s, Wu_s, Wd_s, M, K, N_local, T, C, c->sym_buf, workspace, ws_bytes, d_overflow, algo,
                         stream);
    if (r != SFFN_OK) return r;
    return sffn_allreduce_sym_bf16(c, nullptr, Y, M, K, stream);
}

int sffn_sharded_forward(sffn_comm* c, const void* X, const void* Wg_s, const void* Wu_s, const void* Wd_s, int64_t M,
                         int64_t K, int64_t N_local, int T, int C, void* Y, void* workspace, size_t ws_bytes,
                         uint32_t* d_overflow, int algo, int n_chunks, void* stream) {
    if (!c) return SFFN_ERR_INVALID_ARG;
    if (n_chunks < 1) n_chunks = 1;
    if (M < 0) return SFFN_ERR_SHAPE;
    if (ws_bytes < sffn_forward_workspace_bytes(M, K, N_local, T, C, algo)) return SFFN_ERR_SHAPE;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (n_chunks == 1 || M < 2 * 2048) {
        int r = sffn_forward(X, Wg_s, Wu_s, Wd_s, M, K, N_local, T, C, Y, workspace, ws_bytes, d_overflow, algo,
                             stream);
        if (r != SFFN_OK) return r;
        return sffn_allreduce_bf16(c, Y, M * K, stream);
    }
    if (ensure_events(c, n_chunks) != SFFN_OK) return SFFN_ERR_CUDA;
    // chunk rows rounded to the 2048-row pi windows (P:1078 order per window, reading R21/R24): every chunk starts
    // on a window boundary, so the chunks build exactly the windows and union blocks of one unchunked call
    int64_t rows = (M + n_chunks - 1) / n_chunks;
    rows = (rows + 2047) / 2048 * 2048;
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
