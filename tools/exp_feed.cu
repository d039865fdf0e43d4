// Microbenchmark: per-SM operand feed of the union GEMMs on B200, without the MMAs.
// One persistent CTA per SM walks "tiles" of 64 k-blocks.  Per k-block (one ring stage):
//   A: a 128-row x 64-col bf16 tile of X by TMA (128B swizzle, 16 KB), the same token block for all k-blocks of a tile
//   B: `brows` gathered 128-byte weight-row segments (row = a random unit of the tile, k-slice kb):
//      bmode 0: cp.async.cg 16 B, 8 lanes per row segment (the union kernels' producer mapping)
//      bmode 1: one TMA 2-D box {64, 1} per row (128B swizzle by address), issued by the gather warps' lanes
//      bmode 2: ld.global.v4 to registers + st.shared (LSU round trip) with the stage's mbarrier arrive
//      bmode 4: as 2 with 4 independent 16-byte loads per lane in flight before the stores (batched LSU)
//      bmode 5: 256-bit loads (ld.global.nc.v8, 4 lanes per 128-byte row segment), 4 per lane in flight, 2 x st.shared.v4
// A consumer thread waits for each stage, spins `delay` SM cycles (the MMA time it would take), frees the stage.
// Prints achieved bytes per SM cycle and the stage time.  Not part of the library.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/exp_feed tools/exp_feed.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <random>
#include <algorithm>
#include "../paper_2603_23198_b200/csrc/ptx.cuh"

using namespace sffn;
constexpr int S = 4, KB = 64, ABYTES = 128 * KB * 2, BMAX = 256 * 128;

__device__ __forceinline__ void cp16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_row(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int r) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(r)
        : "memory");
}

struct P {
    int K, ntiles, abytes, brows, bmode, delay, nw, tsplit;
    const uint16_t* W;
    const int* units;   // [ntiles, 256]
    const int* blocks;  // [ntiles]
    int* counter;
    unsigned long long* cycles;
};

__global__ void __launch_bounds__(32 * 26, 1) k_feed(const __grid_constant__ CUtensorMap tX,
                                                      const __grid_constant__ CUtensorMap tW, const P p) {
    extern __shared__ uint8_t sm_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* stA = sm;
    uint8_t* stB = sm + S * ABYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(stB + S * BMAX);
    uint64_t* empty = full + S;
    __shared__ int tiles[1024];
    __shared__ int ntl;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int NW = p.nw;
    const bool lsu_b = p.brows > 0 && p.bmode != 1;  // bmodes 0, 2, 3, 4, 5: every gather thread arrives
    const int tma_rows = p.bmode == 1 ? p.brows : (p.bmode == 3 ? p.brows - p.tsplit : 0);
    const int lsu_rows = p.bmode == 3 ? p.tsplit : p.brows;
    if (threadIdx.x == 0) {
        int n = 0;
        for (int t = blockIdx.x; t < p.ntiles && n < 1024; t += gridDim.x) tiles[n++] = t;  // static: balanced
        ntl = n;
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1 + (lsu_b ? NW * 32 : 0));
            mbar_init(&empty[i], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const long long t0 = clock64();
    const int nt = ntl;
    if (warp == 0) {
        if (lane == 0) {
            int st = 0;
            uint32_t ph = 0;
            for (int i = 0; i < nt; ++i) {
                const int b = p.blocks[tiles[i]];
                for (int kb = 0; kb < p.K / KB; ++kb) {
                    mbar_wait_relaxed(&empty[st], ph ^ 1);
                    const uint32_t tx = p.abytes + tma_rows * 128;
                    if (tx) mbar_arrive_expect_tx(&full[st], tx); else mbar_arrive(&full[st]);
                    if (p.abytes) tma_load_2d(stA + st * ABYTES, &tX, &full[st], kb * KB, b * 128, policy_evict_last());
                    if (++st == S) { st = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            int st = 0;
            uint32_t ph = 0;
            for (int i = 0; i < nt; ++i)
                for (int kb = 0; kb < p.K / KB; ++kb) {
                    mbar_wait_relaxed(&full[st], ph);
                    if (p.delay) {
                        const long long c = clock64();
                        while (clock64() - c < p.delay) {}
                    }
                    mbar_arrive(&empty[st]);
                    if (++st == S) { st = 0; ph ^= 1; }
                }
        }
    } else if (warp >= 2 && warp < 2 + NW && p.brows > 0) {
        const int gw = warp - 2;
        int st = 0;
        uint32_t ph = 0;
        for (int i = 0; i < nt; ++i) {
            const int* u = p.units + static_cast<int64_t>(tiles[i]) * 256;
            for (int kb = 0; kb < p.K / KB; ++kb) {
                mbar_wait_relaxed(&empty[st], ph ^ 1);
                const uint32_t dst = smem_u32(stB + st * BMAX);
                if (p.bmode == 0 || p.bmode == 3) {
                    const int cl = lane & 7, sub = lane >> 3;
                    for (int r = 4 * gw + sub; r < lsu_rows; r += 4 * NW) {
                        const int n = __ldg(u + r);
                        cp16(dst + r * 128 + ((cl ^ (r & 7)) << 4), p.W + static_cast<int64_t>(n) * p.K + kb * KB + 8 * cl);
                    }
                    if (p.bmode == 3)
                        for (int r = lsu_rows + 32 * gw + lane; r < p.brows; r += 32 * NW)
                            tma_row(stB + st * BMAX + r * 128, &tW, &full[st], kb * KB, __ldg(u + r));
                    cp_arrive(&full[st]);
                } else if (p.bmode == 1) {
                    for (int r = 32 * gw + lane; r < p.brows; r += 32 * NW)
                        tma_row(stB + st * BMAX + r * 128, &tW, &full[st], kb * KB, __ldg(u + r));
                } else if (p.bmode == 4) {
                    const int cl = lane & 7, sub = lane >> 3;
                    for (int r0 = 4 * gw + sub; r0 < p.brows; r0 += 16 * NW) {
                        uint4 v[4];
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int r = r0 + 4 * NW * j;
                            if (r < p.brows)
                                v[j] = __ldcg(reinterpret_cast<const uint4*>(p.W + static_cast<int64_t>(__ldg(u + r)) * p.K + kb * KB + 8 * cl));
                        }
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int r = r0 + 4 * NW * j;
                            if (r < p.brows) *reinterpret_cast<uint4*>(stB + st * BMAX + r * 128 + ((cl ^ (r & 7)) << 4)) = v[j];
                        }
                    }
                    mbar_arrive(&full[st]);
                } else if (p.bmode == 5) {
                    const int cl = lane & 3, sub = lane >> 2;
                    for (int r0 = 8 * gw + sub; r0 < p.brows; r0 += 32 * NW) {
                        uint32_t v[4][8];
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int r = r0 + 8 * NW * j;
                            if (r < p.brows) {
                                const uint16_t* src = p.W + static_cast<int64_t>(__ldg(u + r)) * p.K + kb * KB + 16 * cl;
                                asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                                             : "=r"(v[j][0]), "=r"(v[j][1]), "=r"(v[j][2]), "=r"(v[j][3]), "=r"(v[j][4]),
                                               "=r"(v[j][5]), "=r"(v[j][6]), "=r"(v[j][7])
                                             : "l"(src));
                            }
                        }
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int r = r0 + 8 * NW * j;
                            if (r < p.brows) {
                                uint8_t* rb = stB + st * BMAX + r * 128;
                                *reinterpret_cast<uint4*>(rb + (((2 * cl) ^ (r & 7)) << 4)) = make_uint4(v[j][0], v[j][1], v[j][2], v[j][3]);
                                *reinterpret_cast<uint4*>(rb + (((2 * cl + 1) ^ (r & 7)) << 4)) = make_uint4(v[j][4], v[j][5], v[j][6], v[j][7]);
                            }
                        }
                    }
                    mbar_arrive(&full[st]);
                } else {
                    const int cl = lane & 7, sub = lane >> 3;
                    for (int r = 4 * gw + sub; r < p.brows; r += 4 * NW) {
                        const int n = __ldg(u + r);
                        const uint4 v = __ldcg(reinterpret_cast<const uint4*>(p.W + static_cast<int64_t>(n) * p.K + kb * KB + 8 * cl));
                        *reinterpret_cast<uint4*>(stB + st * BMAX + r * 128 + ((cl ^ (r & 7)) << 4)) = v;
                    }
                    mbar_arrive(&full[st]);
                }
                if (++st == S) { st = 0; ph ^= 1; }
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(p.cycles, static_cast<unsigned long long>(clock64() - t0));
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static void tmap(CUtensorMap* m, void* ptr, uint64_t inner, uint64_t outer, uint32_t bi, uint32_t bo) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    cuuint64_t d[2] = {inner, outer}, s[1] = {inner * 2};
    cuuint32_t b[2] = {bi, bo}, e[2] = {1, 1};
    CUresult r = reinterpret_cast<Enc>(f)(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ptr, d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("tmap failed %d\n", r); exit(1); }
}

int main(int argc, char** argv) {
    const int M = 32768, K = 4096, N = 14336;
    const int ntiles = 148 * 24;
    uint16_t *X, *W;
    cudaMalloc(&X, size_t(M) * K * 2);
    cudaMalloc(&W, size_t(N) * K * 2);
    cudaMemset(X, 0, size_t(M) * K * 2);
    cudaMemset(W, 0, size_t(N) * K * 2);
    std::mt19937 rng(1);
    // unit popularity: a 0.365-N "union" per block drawn from a lognormal-weighted pool, 256 units per tile
    std::vector<int> units(size_t(ntiles) * 256), blocks(ntiles);
    // lognormal (sigma 1) unit popularity: concurrently running tiles share hot units, as the real unions do
    std::lognormal_distribution<double> ln(0.0, 1.0);
    std::vector<double> wgt(N);
    for (auto& w : wgt) w = ln(rng);
    std::discrete_distribution<int> pick(wgt.begin(), wgt.end());
    for (int t = 0; t < ntiles; ++t) {
        blocks[t] = t / 20 % 256;
        std::vector<char> used(N, 0);
        std::vector<int> u;
        while ((int)u.size() < 256) { const int n = pick(rng); if (!used[n]) { used[n] = 1; u.push_back(n); } }
        std::sort(u.begin(), u.end());
        std::copy(u.begin(), u.end(), units.begin() + size_t(t) * 256);
    }
    int *du, *db, *cnt;
    unsigned long long* cyc;
    cudaMalloc(&du, units.size() * 4);
    cudaMalloc(&db, blocks.size() * 4);
    cudaMalloc(&cnt, 4);
    cudaMalloc(&cyc, 8);
    cudaMemcpy(du, units.data(), units.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(db, blocks.data(), blocks.size() * 4, cudaMemcpyHostToDevice);
    CUtensorMap tX, tW;
    tmap(&tX, X, K, M, 64, 128);
    tmap(&tW, W, K, N, 64, 1);
    const int smem = 1024 + S * (ABYTES + BMAX) + 256;
    cudaFuncSetAttribute(k_feed, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    struct Cfg { const char* name; int abytes, brows, bmode, delay, nw, tsplit, grid = 0; };
    std::vector<Cfg> cfgs = {
        {"B256 cp.async 8 warps", 0, 256, 0, 0, 8, 0},
        {"B256 cp.async 16 warps", 0, 256, 0, 0, 16, 0},
        {"B256 LSU 16B x1 8 warps", 0, 256, 2, 0, 8, 0},
        {"B256 LSU 16B x4 8 warps", 0, 256, 4, 0, 8, 0},
        {"B256 LSU 16B x4 16 warps", 0, 256, 4, 0, 16, 0},
        {"B256 LSU 32B x4 8 warps", 0, 256, 5, 0, 8, 0},
        {"B256 LSU 32B x4 16 warps", 0, 256, 5, 0, 16, 0},
        {"A + B256 cp.async 8 warps", ABYTES, 256, 0, 0, 8, 0},
        {"A + B256 LSU 16B x4 8 warps", ABYTES, 256, 4, 0, 8, 0},
        {"A + B256 LSU 32B x4 8 warps", ABYTES, 256, 5, 0, 8, 0},
        {"A + B256 LSU 32B x4 16 warps", ABYTES, 256, 5, 0, 16, 0},
        {"A + B128 LSU 32B x4 8 warps", ABYTES, 128, 5, 0, 8, 0},
    };
    if (argc > 1) cfgs.insert(cfgs.end(), {
        {"A + B256 cp.async 16 warps, 148 CTAs", ABYTES, 256, 0, 0, 16, 0, 148},
        {"A + B256 cp.async 16 warps, 74 CTAs", ABYTES, 256, 0, 0, 16, 0, 74},
        {"A + B256 cp.async 16 warps, 37 CTAs", ABYTES, 256, 0, 0, 16, 0, 37},
        {"A + B128 cp.async 16 warps, 74 CTAs", ABYTES, 128, 0, 0, 16, 0, 74},
        {"A only, 74 CTAs", ABYTES, 0, 0, 0, 8, 0, 74},
        {"B256 cp.async 16 warps, 74 CTAs", 0, 256, 0, 0, 16, 0, 74},
        {"A only (TMA 16 KB)", ABYTES, 0, 0, 0, 8, 0},
        {"B256 cp.async 4 warps", 0, 256, 0, 0, 4, 0},
        {"B256 cp.async 8 warps", 0, 256, 0, 0, 8, 0},
        {"B256 cp.async 12 warps", 0, 256, 0, 0, 12, 0},
        {"B256 cp.async 16 warps", 0, 256, 0, 0, 16, 0},
        {"B256 cp.async 24 warps", 0, 256, 0, 0, 24, 0},
        {"B256 TMA box{64,1} 8 warps", 0, 256, 1, 0, 8, 0},
        {"B256 cp.async 192 + TMA 64, 8 warps", 0, 256, 3, 0, 8, 192},
        {"B256 cp.async 160 + TMA 96, 8 warps", 0, 256, 3, 0, 8, 160},
        {"B256 cp.async 192 + TMA 64, 16 warps", 0, 256, 3, 0, 16, 192},
        {"A + B256 cp.async 8 warps", ABYTES, 256, 0, 0, 8, 0},
        {"A + B256 cp.async 16 warps", ABYTES, 256, 0, 0, 16, 0},
        {"A + B256 cp.async 192 + TMA 64, 16 w", ABYTES, 256, 3, 0, 16, 192},
        {"A + B128 cp.async 8 warps", ABYTES, 128, 0, 0, 8, 0},
        {"A + B128 cp.async 16 warps", ABYTES, 128, 0, 0, 16, 0},
        {"A + B128 cp.async 96 + TMA 32, 16 w", ABYTES, 128, 3, 0, 16, 96},
        {"A + B128 cp.async 16 w, delay 512", ABYTES, 128, 0, 512, 16, 0},
        {"A + B256 cp.async 16 w, delay 512", ABYTES, 256, 0, 512, 16, 0},
    });
    for (auto& c : cfgs) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaMemset(cnt, 0, 4);
            cudaMemset(cyc, 0, 8);
            P p{K, ntiles, c.abytes, c.brows, c.bmode, c.delay, c.nw, c.tsplit, W, du, db, cnt, cyc};
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            const int g = c.grid ? c.grid : sms;
            k_feed<<<g, 32 * (2 + c.nw), smem>>>(tX, tW, p);
            cudaEventRecord(e1);
            cudaError_t err = cudaEventSynchronize(e1);
            if (err != cudaSuccess) { printf("%s: %s\n", c.name, cudaGetErrorString(err)); return 1; }
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            unsigned long long cy;
            cudaMemcpy(&cy, cyc, 8, cudaMemcpyDeviceToHost);
            const double stages = double(ntiles) * (K / KB);
            const double bytes = stages * (c.abytes + c.brows * 128.0);
            const double avg_cyc = double(cy) / g;  // cycles per CTA
            if (rep == 1)
                printf("%-40s %8.3f ms  %7.1f TB/s  %6.1f B/cyc/SM  %6.0f cyc/stage  (CTA-avg clk %.0f MHz)\n", c.name, ms,
                       bytes / ms / 1e9, bytes / g / avg_cyc, avg_cyc / (stages / g), avg_cyc / ms / 1e3);
        }
    }
    return 0;
}
