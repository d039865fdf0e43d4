// Microbenchmark: per-SM throughput of gathering random 128-byte row segments into SMEM on B200.
//   mode 0: cp.async.cg 16 B (NW warps, 8 lanes per row segment)
//   mode 1: TMA tile::gather4 (box {64 bf16, 1 row}, 128B swizzle), issued by one thread
//   mode 2: both: cp.async for 256 - R rows, gather4 for R rows per "k-block"
// Each CTA (one per SM) loops over ITERS k-blocks; a k-block = 256 rows x 128 B = 32 KB into a 4-stage ring.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/exp_gather_bw tools/exp_gather_bw.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include "../paper_2603_23198_b200/csrc/ptx.cuh"

using namespace sffn;
constexpr int STAGES = 4, ROWS = 256, SEG = 128, KB_BYTES = ROWS * SEG;

__device__ __forceinline__ void cp16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void g4(void* dst, const CUtensorMap* m, uint64_t* bar, int c, int r0, int r1, int r2, int r3) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)),
                 "r"(smem_u32(bar)), "r"(c), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
                 : "memory");
}

template <int NW>
__global__ void __launch_bounds__(32 * (NW + 1), 1)
    k_gather(const __grid_constant__ CUtensorMap tm, const uint16_t* __restrict__ W, const int* __restrict__ idx, int K,
             int iters, int R /* rows via TMA */, int mode) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* buf = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(buf + STAGES * KB_BYTES);
    uint64_t* empty = full + STAGES;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int lsu_rows = mode == 1 ? 0 : (mode == 0 ? ROWS : ROWS - R);
    const int tma_rows = ROWS - lsu_rows;
    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&full[i], 1 + NW * 32);
            mbar_init(&empty[i], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int* ib = idx + static_cast<int64_t>(blockIdx.x) * iters * ROWS;
    if (warp < NW) {
        // rows r = 4 warp + sub + 4 NW i; indices for k-block it+1 are loaded while k-block it is issued
        constexpr int NP = (ROWS + 4 * NW - 1) / (4 * NW);
        const int c8 = lane & 7, sub = lane >> 3;
        int stage = 0;
        uint32_t phase = 0;
        int cur[NP], nxt[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) {
            const int r = 4 * warp + sub + 4 * NW * i;
            cur[i] = r < lsu_rows ? __ldg(ib + r) : 0;
        }
        for (int it = 0; it < iters; ++it) {
            const int itn = it + 1 < iters ? it + 1 : it;
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                const int r = 4 * warp + sub + 4 * NW * i;
                nxt[i] = r < lsu_rows ? __ldg(ib + itn * ROWS + r) : 0;
            }
            mbar_wait(&empty[stage], phase ^ 1);
            const uint32_t dst = smem_u32(buf + stage * KB_BYTES);
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                const int r = 4 * warp + sub + 4 * NW * i;
                if (r < lsu_rows)
                    cp16(dst + r * SEG + ((c8 ^ (r & 7)) << 4),
                         W + static_cast<int64_t>(cur[i]) * K + (it % (K / 64)) * 64 + 8 * c8);
            }
            cp_arrive(&full[stage]);
#pragma unroll
            for (int i = 0; i < NP; ++i) cur[i] = nxt[i];
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
    } else if (lane == 0) {
        // TMA issuer (indices staged in SMEM one k-block ahead by lane 0) + consumer bookkeeping
        int stage = 0, cstage = 0;
        uint32_t phase = 0, cphase = 0;
        for (int it = 0; it < iters; ++it) {
            int ids[64];
#pragma unroll
            for (int j = 0; j < 64; ++j) ids[j] = (lsu_rows + j < ROWS) ? __ldg(ib + it * ROWS + lsu_rows + j) : 0;
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_arrive_expect_tx(&full[stage], tma_rows * SEG);
#pragma unroll
            for (int j = 0; j < 64; j += 4)
                if (lsu_rows + j < ROWS)
                    g4(buf + stage * KB_BYTES + (lsu_rows + j) * SEG, &tm, &full[stage], (it % (K / 64)) * 64, ids[j],
                       ids[j + 1], ids[j + 2], ids[j + 3]);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
            if (it >= STAGES - 2) {
                mbar_wait(&full[cstage], cphase);
                mbar_arrive(&empty[cstage]);
                if (++cstage == STAGES) { cstage = 0; cphase ^= 1; }
            }
        }
        while (cstage != stage || cphase != phase) {
            mbar_wait(&full[cstage], cphase);
            mbar_arrive(&empty[cstage]);
            if (++cstage == STAGES) { cstage = 0; cphase ^= 1; }
        }
    }
}

typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int NW>
float run(CUtensorMap tm, uint16_t* W, int* idx, int K, int iters, int R, int mode, int sms) {
    auto kern = k_gather<NW>;
    const int smem = STAGES * KB_BYTES + 1024 + 256;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    kern<<<sms, 32 * (NW + 1), smem>>>(tm, W, idx, K, iters, R, mode);
    cudaEventRecord(a);
    kern<<<sms, 32 * (NW + 1), smem>>>(tm, W, idx, K, iters, R, mode);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

int main() {
    const int N = 14336, K = 4096, iters = 400, sms = 148;
    uint16_t* W;
    int* idx;
    cudaMalloc(&W, static_cast<size_t>(N) * K * 2);
    cudaMemset(W, 1, static_cast<size_t>(N) * K * 2);
    std::vector<int> h(static_cast<size_t>(sms) * iters * ROWS);
    std::mt19937 rng(1);
    for (auto& x : h) x = rng() % N;
    cudaMalloc(&idx, h.size() * 4);
    cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    void* p;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)N};
    cuuint64_t str[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {64, 1};
    cuuint32_t es[2] = {1, 1};
    ((PFN)p)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, W, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const double bytes = static_cast<double>(sms) * iters * KB_BYTES;
    auto rep = [&](const char* name, float ms) {
        const double bps = bytes / (ms * 1e-3);
        printf("%-28s %8.3f ms  %7.2f TB/s  %6.1f B/cycle/SM @1.9GHz  (%.0f cycles per 32 KB k-block)\n", name, ms,
               bps / 1e12, bps / sms / 1.9e9, KB_BYTES / (bps / sms / 1.9e9));
    };
    rep("cp.async 4 warps", run<4>(tm, W, idx, K, iters, 0, 0, sms));
    rep("cp.async 8 warps", run<8>(tm, W, idx, K, iters, 0, 0, sms));
    rep("cp.async 16 warps", run<16>(tm, W, idx, K, iters, 0, 0, sms));
    rep("1 cp.async warp + gather4 64", run<1>(tm, W, idx, K, iters, 64, 2, sms));
    for (int R : {16, 32, 48, 64}) {
        char nm[64];
        snprintf(nm, sizeof nm, "8 warps + gather4 %d rows", R);
        rep(nm, run<8>(tm, W, idx, K, iters, R, 2, sms));
    }
    return 0;
}
