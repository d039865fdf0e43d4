// gemm_union.cuh — tensor-core sparse up/down over per-block neuron unions.
//
// Eq.3 regrouped: for a block b of 128 token rows and U_b = union of their active neurons,
//   H_b = G_b ⊙ (X_b · W_u[U_b]^T)        (UP kernel;  G_b = TwELL gate values scattered into U_b
//                                           coordinates, 0 where (m, n) is not stored)
//   Y_b = H_b · W_d[U_b, :]               (DOWN kernel)
// Every term skipped relative to Eq.1 has h_g = 0, exactly as in Alg.2; the terms computed
// with G = 0 add exact zeros.  Both kernels are persistent warp-specialized tcgen05 GEMMs like
// gemm_tc.cuh; the dense A operand comes by TMA, the weight rows of U_b are gathered by four producer
// warps with 16-byte cp.async.cg into the 128-byte-swizzled UMMA layout (TMA tile::gather4 measured
// ~70 SM cycles per instruction on B200 — 8x too slow to feed the tensor cores, tools/exp_gather4.cu):
//   UP   B operand: W_u[U_b[256c + r], k0:k0+64]       K-major
//   DOWN B operand: W_d[U_b[k0 + r], 256j:256j+256]     MN-major (4 x 64-column atoms)
// cp.async completion is signalled with cp.async.mbarrier.arrive.noinc on the stage's full barrier.
#pragma once
#include "gemm_tc.cuh"
#include "union.cuh"

namespace sffn {

typedef unsigned short bf16_t;

struct UnionArgs {
    int M, K, N, T, C;
    int NB;             // token blocks of 128
    int NJ;             // DOWN: output column tiles of 256
    int group;          // DOWN: token blocks per raster group
    const uint32_t* tw;  // UP: packed TwELL [M, N/C]
    UnionMeta um;
    const bf16_t* wsrc;  // UP: W_u, DOWN: W_d, both [N, K]
    const int32_t* perm;  // DOWN: output row of permuted row i
    int* counter;         // dynamic tile scheduler (zeroed by union_scan_kernel)
    bf16_t* Y;            // DOWN: output [M, K]
    // DOWN with the fused window-granular all-reduce (NEXT-3, sffn_sharded_forward_fused); Y = this rank's
    // symmetric window.  ptrs[p] = rank p's window base (LSA, P2P-mapped), ptrs[G] = its multicast address or 0.
    const uint64_t* ptrs;
    int G, rank;
};

// ---------------------------------------------------------------- fused all-reduce helpers (NEXT-3)
constexpr int FUSE_WIN = 2048;
constexpr int FUSE_WARPS = 2;  // reducer warps: 2 (idle after the TMEM allocation) and 3
constexpr int FUSE_U = 8;      // 16-byte loads in flight per reducer lane  // rows per reduction window (= the pi window: a DOWN raster group of 16 blocks)
__device__ __forceinline__ uint32_t ld_relaxed_sys_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fuse_bf16x8_acc(float (&a)[8], const uint4& v) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        a[2 * i] += __uint_as_float(w[i] << 16);
        a[2 * i + 1] += __uint_as_float(w[i] & 0xFFFF0000u);
    }
}

// 16-byte cp.async of a gathered weight-row segment (L2 only: .cg); src_bytes < 16 zero-fills the rest
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
#ifndef SFFN_UG_NOGATHER  // timing probe only (tools): gathers skipped, results wrong
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
#endif
}
// UP gathers (row-major W_u: the row's next k-block is the next 128 bytes): optional L2 prefetch-size hint
#ifndef SFFN_UP_L2PF
#define SFFN_UP_L2PF 0
#endif
__device__ __forceinline__ void cp_async16_up(uint32_t dst, const void* src) {
#ifndef SFFN_UG_NOGATHER
#if SFFN_UP_L2PF == 256
    asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
#elif SFFN_UP_L2PF == 128
    asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
#else
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
#endif
#endif
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}


// MN-major operand, 128-byte swizzle: 64-element MN atoms LBO apart, 8-row K groups SBO apart.
__device__ __forceinline__ uint64_t umma_desc_sw128_mn(uint32_t smem_addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((smem_addr & 0x3FFFFu) >> 4);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(2) << 61;
    return d;
}

__device__ __forceinline__ int upper_bound_i32(const int32_t* a, int n, int key) {  // first i with a[i] > key
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(a + mid) <= key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// byte offset of element (r, c) in a [32 rows x 64 bf16] 128B-swizzled TMA box (1024-aligned base)
__device__ __forceinline__ uint32_t sw128_off(int r, int c) {
    return static_cast<uint32_t>(r * 128 + ((((c >> 3) ^ r) & 7) << 4) + ((c & 7) << 1));
}

// k-block of the union GEMMs.  64 (default): 128-byte K-major rows (SWIZZLE_128B), 4 stages of 48 KB.  32: 64-byte
// rows (SWIZZLE_64B), 8 stages of 24 KB in the same shared memory (more, smaller stages in flight) — measured
// 1.30x (UP) and 1.67x (DOWN) SLOWER on the 7B step (CUPTI, two alternating rounds): the per-stage costs (barrier
// round trips, MMA issue, twice the gather instructions per byte) dominate; kept as a compile-time option.
#ifndef SFFN_UG_BK
#define SFFN_UG_BK 64
#endif
constexpr int UG_BK = SFFN_UG_BK;
static_assert(UG_BK == 32 || UG_BK == 64, "union k-block is 32 or 64");
constexpr int UG_A_BYTES = GEMM_BM * UG_BK * 2;           // A tile: 128 rows x UG_BK
constexpr int UG_B_BYTES = 256 * UG_BK * 2;               // B tile: 256 (UP: rows, DOWN: columns) x UG_BK
constexpr int UG_STAGE_BYTES = UG_A_BYTES + UG_B_BYTES;
constexpr int UG_STAGES = UG_BK == 32 ? 8 : 4;
constexpr int UG_ROWB = UG_BK * 2;                        // bytes of one K-major row segment = the swizzle span
// K-major operand descriptor for the UG_BK layout: SWIZZLE_64B (8-row atoms of 512 B, layout type 4) or
// SWIZZLE_128B (8-row atoms of 1 KB, layout type 2); LBO unused for swizzled K-major
__device__ __forceinline__ uint64_t umma_desc_ug(uint32_t smem_addr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((smem_addr & 0x3FFFFu) >> 4);
    d |= static_cast<uint64_t>(1) << 16;
    d |= static_cast<uint64_t>((8 * UG_ROWB) >> 4) << 32;  // SBO: 8 rows
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(UG_BK == 32 ? 4 : 2) << 61;
    return d;
}
// 16-byte chunk c of K-major row r in the UG_BK swizzled layout (TMA SWIZZLE_64B / 128B pattern)
__device__ __forceinline__ uint32_t ug_kmajor_off(int r, int c) {
    return static_cast<uint32_t>(r * UG_ROWB + ((c ^ (UG_BK == 32 ? ((r >> 1) & 3) : (r & 7))) << 4));
}
constexpr int UG_GPRE = 8;  // UP epilogue: gate entries per row prefetched before the accumulator wait
#ifndef UG_NGW
#define UG_NGW 8
#endif
constexpr int UG_GW = UG_NGW;                  // gather producer warps (8..8+UG_GW-1)
constexpr int UG_THREADS = 256 + 32 * UG_GW;   // warps 0-7 as gemm_tc + gather producer warps
constexpr int UG_GATHER = 32 * UG_GW;
constexpr int UG_EWB = 8192;  // epilogue staging per warp
constexpr int UG_SMEM = 1024 + UG_STAGES * UG_STAGE_BYTES + 4 * UG_EWB + 1024;
constexpr int UG_RING = 8;       // tile-scheduler ring depth
constexpr int UG_READERS = UG_GW + 5;  // gather warps + MMA thread + 4 epilogue warps (pair kernels)
// Epilogue warp groups of the single-CTA union GEMMs: with 2, warps 4-7 drain columns 0-127 of an accumulator and
// warps 8+UG_GW..+3 columns 128-255 at the same time (4 KB of staging each, 64-column passes): the epilogue takes
// half as long.  At K = 2048 (1B) one group's UP epilogue was slower than a tile's mainloop: without the gathers the
// MMA thread spent its time waiting for the accumulator (ncu, tools/prof_union_src.sh).  The fused all-reduce DOWN
// (which counts 4 epilogue arrivals per tile at the window owner) keeps one group.
#ifndef SFFN_UG_EPI_GROUPS
#define SFFN_UG_EPI_GROUPS 2
#endif
constexpr int UG_EG = SFFN_UG_EPI_GROUPS;
static_assert(UG_EG == 1 || UG_EG == 2, "1 or 2 epilogue groups");
constexpr int UG_THREADS2 = UG_THREADS + 128 * (UG_EG - 1);  // single-CTA (non-fused) union GEMMs

template <bool UP, bool FUSED = false>
__global__ void __launch_bounds__(FUSED ? UG_THREADS : UG_THREADS2, 1)
    union_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmOut, const UnionArgs args) {
    constexpr int S = UG_STAGES;
    constexpr int EG = FUSED ? 1 : UG_EG;        // epilogue warp groups (column halves)
    constexpr int EWB = UG_EWB / EG;             // staging bytes per epilogue warp
    constexpr int PC = EWB / 64;                 // columns per staging pass (32 rows x PC bf16 = EWB bytes)
    constexpr int GC = 256 / EG;                 // columns per group
    constexpr int READERS = UG_GW + 1 + 4 * EG;  // gather warps + MMA thread + epilogue warps
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* stA = smem;
    uint8_t* stB = smem + S * UG_A_BYTES;
    uint8_t* epi = stB + S * UG_B_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(epi + 4 * UG_EWB);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    uint64_t* tempty = tfull + 2;
    uint64_t* gbar = tempty + 2;  // [4] epilogue: G tile loaded
    uint64_t* sfull = gbar + 4;   // [UG_RING] tile ring
    uint64_t* sempty = sfull + UG_RING;
    int* sched = reinterpret_cast<int*>(sempty + UG_RING);  // [UG_RING]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sched + UG_RING);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int N = args.N;
    const int NB = args.NB;
    const int num_tiles = UP ? __ldg(args.um.chunk_off) : NB * args.NJ;
    const int nk_up = (args.K + UG_BK - 1) / UG_BK;

    if (threadIdx.x == 0) {
        tma_prefetch(&tmA);
        tma_prefetch(&tmB);
        tma_prefetch(&tmOut);
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1 + UG_GATHER);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4 * EG);
        }
        for (int i = 0; i < 4; ++i) mbar_init(&gbar[i], 1);
        for (int i = 0; i < UG_RING; ++i) {
            mbar_init(&sfull[i], 1);
            mbar_init(&sempty[i], READERS);
        }
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    // dynamic scheduler ring: warp 0 lane 0 claims tiles (atomicAdd) in the raster order and publishes them;
    // every role reads the same sequence.  next_tile() returns -1 when the work is exhausted.
    auto next_tile = [&](int& ridx, uint32_t& rphase, bool arrive_lane) -> int {
        mbar_wait(&sfull[ridx], rphase);
        const int t = *reinterpret_cast<volatile int*>(&sched[ridx]);
        if (arrive_lane) mbar_arrive(&sempty[ridx]);
        if (++ridx == UG_RING) {
            ridx = 0;
            rphase ^= 1;
        }
        return t;
    };

    // tile -> (b, c | j, rows/len)
    auto tile_info = [&](int tile, int& b, int& cj, int& len) {
        if (UP) {
            const int v = __ldg(args.um.tiles + tile);
            b = v >> 8;
            cj = v & 255;
            len = min(256, __ldg(args.um.ulen + b) - 256 * cj);  // rows of this chunk (multiple of 64)
        } else {
            // grouped raster: args.group blocks sweep all output column tiles together (L2 working set)
            const int G = args.group;
            const int per = G * args.NJ;
            const int grp = tile / per;
            const int gb = min(G, NB - grp * G);
            const int in = tile - grp * per;
            b = grp * G + in % gb;
            cj = in / gb;
            len = __ldg(args.um.ulen + b);  // reduction length (multiple of 64)
        }
    };

    if (warp == 0) {
        // ------------------------------------------------------------ A operand by TMA (one thread)
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int widx = 0;
            uint32_t wphase = 0;
            for (;;) {
                mbar_wait(&sempty[widx], wphase ^ 1);
                int tile = atomicAdd(args.counter, 1);
                if (tile >= num_tiles) tile = -1;
                sched[widx] = tile;
                mbar_arrive(&sfull[widx]);
                if (++widx == UG_RING) {
                    widx = 0;
                    wphase ^= 1;
                }
                if (tile < 0) break;
                int b, cj, len;
                tile_info(tile, b, cj, len);
                const int nk = UP ? nk_up : len / UG_BK;
                // dense block (union forced to all N units by the prep kernel): B by TMA tiles, no gathers
                const bool dense = __ldg(args.um.udense + b) != 0;
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait_relaxed(&empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&full[stage], dense ? UG_STAGE_BYTES : UG_A_BYTES);
                    tma_load_2d(stA + stage * UG_A_BYTES, &tmA, &full[stage], kb * UG_BK, b * GEMM_BM,
                                policy_evict_last());
                    if (dense) {
                        uint8_t* bdst = stB + stage * UG_B_BYTES;
                        if (UP) {  // W_u rows [256 cj, 256 cj + 256), k-slice kb: K-major box {UG_BK, 256}
                            tma_load_2d(bdst, &tmB, &full[stage], kb * UG_BK, 256 * cj, policy_evict_last());
                        } else {   // W_d rows [UG_BK kb, +UG_BK), columns 256 cj + 64 q: four MN-major {64, UG_BK} atoms
#pragma unroll
                            for (int q = 0; q < 4; ++q)
                                tma_load_2d(bdst + q * (UG_B_BYTES / 4), &tmB, &full[stage], 256 * cj + 64 * q,
                                            kb * UG_BK, policy_evict_last());
                        }
                    }
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp >= 8 && warp < 8 + UG_GW) {
        // ------------------------------------------------------------ B operand: gathered weight rows
        // UP (K-major): LPR consecutive lanes copy one UG_ROWB-byte row segment (16 B each), RPI rows per warp
        // instruction; DOWN (MN-major, 128-byte swizzle): one neuron row's 4 adjacent 64-column atoms (512 B) per
        // warp instruction.  Every warp instruction moves whole row segments.
        const int gw = warp - 8;          // 0..UG_GW-1
        int stage = 0;
        uint32_t phase = 0;
        int ridx = 0;
        uint32_t rphase = 0;
        for (;;) {
            const int tile = next_tile(ridx, rphase, lane == 0);
            if (tile < 0) break;
            int b, cj, len;
            tile_info(tile, b, cj, len);
            const int32_t* ul = args.um.ulist + static_cast<int64_t>(b) * N;
            if (__ldg(args.um.udense + b) != 0) {
                // dense block: B comes by TMA (warp 0); keep the per-stage arrivals of the full barrier
                const int nk = UP ? nk_up : len / UG_BK;
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait_relaxed(&empty[stage], phase ^ 1);
                    cp_async_arrive_noinc(&full[stage]);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            } else if (UP) {
                constexpr int LPR = UG_BK / 8;             // lanes per row segment
                constexpr int RPI = 32 / LPR;              // rows per warp instruction
                constexpr int NP = 256 / (RPI * UG_GW);    // instructions per warp per stage
                const int cl = lane % LPR, sub = lane / LPR;
                int nidx[NP];
#pragma unroll
                for (int i = 0; i < NP; ++i) {
                    const int r = RPI * UG_GW * i + RPI * gw + sub;
                    nidx[i] = r < len ? __ldg(ul + 256 * cj + r) : -1;
                }
                for (int kb = 0; kb < nk_up; ++kb) {
                    mbar_wait_relaxed(&empty[stage], phase ^ 1);
                    const uint32_t dst = smem_u32(stB + stage * UG_B_BYTES);
#pragma unroll
                    for (int i = 0; i < NP; ++i) {
                        const int r = RPI * UG_GW * i + RPI * gw + sub;
                        if (nidx[i] >= 0)
                            cp_async16_up(dst + ug_kmajor_off(r, cl),
                                          args.wsrc + static_cast<int64_t>(nidx[i]) * args.K + kb * UG_BK + 8 * cl);
                    }
                    cp_async_arrive_noinc(&full[stage]);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            } else {
                // pass i covers k-block row r = UG_GW i + gw, MN atom a = sub (columns 256 cj + 64 a + 8 c8)
                constexpr int NP = UG_BK / UG_GW;
                const int c8 = lane & 7, sub = lane >> 3;
                const int nk = len / UG_BK;
                const int col = cj * 256 + sub * 64 + 8 * c8;
                const bool in = col < args.K;
                // union indices two k-blocks ahead (an L2 round trip is about one k-block of MMA time), issued before
                // the stage wait so their latency overlaps it.  (A compile-time register ring 2-4 k-blocks ahead,
                // which never copies a pending load, measured 8% slower: DOWN 1195 vs 1105 us, CUPTI, two rounds.)
                int nidx[NP], n1[NP];
#pragma unroll
                for (int i = 0; i < NP; ++i) {
                    nidx[i] = __ldg(ul + UG_GW * i + gw);
                    n1[i] = __ldg(ul + (nk > 1 ? UG_BK : 0) + UG_GW * i + gw);
                }
                for (int kb = 0; kb < nk; ++kb) {
                    int nxt[NP];
                    const int kn = kb + 2 < nk ? kb + 2 : nk - 1;
#pragma unroll
                    for (int i = 0; i < NP; ++i) nxt[i] = __ldg(ul + kn * UG_BK + UG_GW * i + gw);
                    mbar_wait_relaxed(&empty[stage], phase ^ 1);
                    const uint32_t dst = smem_u32(stB + stage * UG_B_BYTES) + sub * (UG_B_BYTES / 4);
#pragma unroll
                    for (int i = 0; i < NP; ++i) {
                        const int r = UG_GW * i + gw;
                        cp_async16(dst + r * 128 + ((c8 ^ (r & 7)) << 4),
                                   args.wsrc + static_cast<int64_t>(nidx[i]) * args.K + (in ? col : 0), in ? 16 : 0);
                    }
                    cp_async_arrive_noinc(&full[stage]);
#pragma unroll
                    for (int i = 0; i < NP; ++i) {
                        nidx[i] = n1[i];
                        n1[i] = nxt[i];
                    }
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            int ridx = 0;
            uint32_t rphase = 0;
            for (;;) {
                const int tile = next_tile(ridx, rphase, true);
                if (tile < 0) break;
                int b, cj, len;
                tile_info(tile, b, cj, len);
                const int nk = UP ? nk_up : len / UG_BK;
                const uint32_t idesc = UP ? umma_idesc_bf16(GEMM_BM, len) : (umma_idesc_bf16(GEMM_BM, 256) | (1u << 16));
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + static_cast<uint32_t>(acc * GEMM_BN);
                for (int kb = 0; kb < nk; ++kb) {
                    // relaxed per-stage wait (an acquire wait invalidates the SM's L1 every k-block, hurting the
                    // gather warps' index loads); the cp.async data is complete when the stage's barrier flips
                    mbar_wait_relaxed(&full[stage], phase);
                    fence_async_smem();  // cp.async (generic proxy) writes -> tensor-core reads (async proxy)
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(stA + stage * UG_A_BYTES);
                    const uint32_t b0 = smem_u32(stB + stage * UG_B_BYTES);
#pragma unroll
                    for (int k = 0; k < UG_BK / 16; ++k) {
                        // DOWN B: MN-major atoms of UG_BK k-rows x 128 B (LBO = atom size), 8-row groups 1 KB apart
                        const uint64_t bd = UP ? umma_desc_ug(b0 + k * 32)
                                               : umma_desc_sw128_mn(b0 + k * 2048, UG_B_BYTES / 4, 1024);
                        umma_f16(d, umma_desc_ug(a0 + k * 32), bd, idesc, (kb | k) != 0);
                    }
                    umma_commit(&empty[stage]);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma_commit(&tfull[acc]);
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else if (FUSED && !UP && warp >= 4 - FUSE_WARPS && warp < 4) {
        // ------------------------------------------------------------ fused all-reduce (window granular)
        // Windows owned by this rank (w % G == rank), in raster order: wait until every rank's epilogue warps have
        // counted all their tiles of the window (4 per block and column tile), then this CTA reduces its slice of
        // the window's rows across the ranks' windows (multimem.ld_reduce + multimem.st through the switch, else
        // P2P loads, fp32 sum, P2P stores into every window) — while later windows are still being computed.
        const int nwin = (args.M + FUSE_WIN - 1) / FUSE_WIN;
        const int64_t K8 = args.K / 8;
        const int rpc = (FUSE_WIN + gridDim.x - 1) / gridDim.x;  // rows of a window per CTA
        const uint32_t* flags = reinterpret_cast<const uint32_t*>(args.ptrs[args.rank] + args.ptrs[args.G + 1]);
        const uint64_t mc = args.ptrs[args.G];
        const int rl = (warp - (4 - FUSE_WARPS)) * 32 + lane;  // reducer lane
        for (int w = args.rank; w < nwin; w += args.G) {
            const int rows_w = min(FUSE_WIN, args.M - w * FUSE_WIN);
            const int blocks = (rows_w + GEMM_BM - 1) / GEMM_BM;
            const uint32_t target = static_cast<uint32_t>(4 * blocks * args.NJ * args.G);
            // one poller per CTA (relaxed loads: an acquire load per poll would invalidate L1 each time under the
            // running GEMM), one acquire fence on success, then a named barrier releases the reducer warps
            if (rl == 0) {
                long long spins = 0;
                uint32_t v;
                while (static_cast<int32_t>((v = ld_relaxed_sys_u32(flags + w)) - target) < 0) {
                    __nanosleep(500);
                    if (++spins == (1ll << 27)) {  // > 1 min: a rank is gone; fail the launch instead of hanging
                        printf("sffn fused: cta %d window %d counter %u target %u\n", blockIdx.x, w, v, target);
                        __trap();
                    }
                }
                asm volatile("fence.acq_rel.sys;" ::: "memory");
            }
            asm volatile("bar.sync 1, %0;" ::"n"(32 * FUSE_WARPS) : "memory");
            const int r0 = w * FUSE_WIN + blockIdx.x * rpc;
            const int r1 = min(w * FUSE_WIN + rows_w, r0 + rpc);
            if (r1 <= r0) continue;
            const int64_t q0 = static_cast<int64_t>(r0) * K8, q1 = static_cast<int64_t>(r1) * K8;
            // FUSE_U independent 16-byte loads in flight per lane before the stores (one or two warps per SM)
            for (int64_t qb = q0 + rl; qb < q1; qb += FUSE_U * 32 * FUSE_WARPS) {
                if (mc) {
                    uint4 v[FUSE_U];
#pragma unroll
                    for (int u = 0; u < FUSE_U; ++u) {
                        const int64_t q = qb + u * 32 * FUSE_WARPS;
                        if (q < q1)
                            asm volatile(
                                "multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                                : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                                : "l"(reinterpret_cast<uint4*>(mc) + q)
                                : "memory");
                    }
#pragma unroll
                    for (int u = 0; u < FUSE_U; ++u) {
                        const int64_t q = qb + u * 32 * FUSE_WARPS;
                        if (q < q1)
                            asm volatile("multimem.st.relaxed.sys.global.v4.bf16x2 [%0], {%1,%2,%3,%4};" ::"l"(
                                             reinterpret_cast<uint4*>(mc) + q),
                                         "r"(v[u].x), "r"(v[u].y), "r"(v[u].z), "r"(v[u].w)
                                         : "memory");
                    }
                } else {
                    float acc8[FUSE_U][8];
#pragma unroll
                    for (int u = 0; u < FUSE_U; ++u)
#pragma unroll
                        for (int i = 0; i < 8; ++i) acc8[u][i] = 0.f;
                    for (int p = 0; p < args.G; ++p) {
                        const uint4* src = reinterpret_cast<const uint4*>(args.ptrs[p]);
                        uint4 v[FUSE_U];
#pragma unroll
                        for (int u = 0; u < FUSE_U; ++u) {
                            const int64_t q = qb + u * 32 * FUSE_WARPS;
                            v[u] = q < q1 ? __ldcv(src + q) : make_uint4(0, 0, 0, 0);
                        }
#pragma unroll
                        for (int u = 0; u < FUSE_U; ++u) fuse_bf16x8_acc(acc8[u], v[u]);
                    }
#pragma unroll
                    for (int u = 0; u < FUSE_U; ++u) {
                        const int64_t q = qb + u * 32 * FUSE_WARPS;
                        if (q < q1) {
                            const uint4 o = make_uint4(pack_bf16x2(acc8[u][0], acc8[u][1]),
                                                       pack_bf16x2(acc8[u][2], acc8[u][3]),
                                                       pack_bf16x2(acc8[u][4], acc8[u][5]),
                                                       pack_bf16x2(acc8[u][6], acc8[u][7]));
                            for (int p = 0; p < args.G; ++p) reinterpret_cast<uint4*>(args.ptrs[p])[q] = o;
                        }
                    }
                }
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------------------------ epilogue (EG groups of 4 warps)
        const int ew = warp & 3;                   // TMEM lane quarter: a warp reads lanes 32 (warp % 4) .. + 31
        const int eg = warp >= 8 ? 1 : 0;          // column half (EG = 2)
        const int g0 = eg * GC;                    // first accumulator column of this group
        uint8_t* stg = epi + (eg * 4 + ew) * EWB;
        int acc = 0;
        uint32_t acc_phase = 0;
        int ridx = 0;
        uint32_t rphase = 0;
        for (;;) {
            const int tile = next_tile(ridx, rphase, lane == 0);
            if (tile < 0) break;
            int b, cj, len;
            tile_info(tile, b, cj, len);
            const int row0 = b * GEMM_BM + ew * 32;
            // UP: this row's gate entries of the chunk, loaded before waiting for the accumulator
            int e0 = 0, e1 = 0;
            const uint32_t* gl = nullptr;
            uint32_t gpre[UG_GPRE];
            // dense block (identity union, position = unit): the gates come straight from the row's TwELL tiles of
            // this chunk (no gate list is built for dense blocks)
            const bool dense_blk = UP && __ldg(args.um.udense + b) != 0;
            const uint32_t* twrow = nullptr;
            if constexpr (UP) {
                const int64_t prow = static_cast<int64_t>(row0) + lane;  // pi-ordered row (H_c row)
                if (dense_blk) {
                    if (prow < args.M) twrow = args.tw + static_cast<int64_t>(__ldg(args.perm + prow)) * (N / args.C);
                } else {
                    gl = args.um.glist + prow * args.um.lmax;
                    const uint16_t* co = args.um.coff + prow * (args.um.nchunk + 1);
                    e0 = __ldg(co + cj);
                    e1 = __ldg(co + cj + 1);
#pragma unroll
                    for (int i = 0; i < UG_GPRE; ++i) gpre[i] = e0 + i < e1 ? __ldg(gl + e0 + i) : 0u;
                }
            }
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const uint32_t tb = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + static_cast<uint32_t>(acc * GEMM_BN);
            if constexpr (UP) {
                // staging <- this row's gate values for the chunk (from the compact gate list, zero elsewhere),
                // then H = G * (X W_u^T) in place, then TMA store of the H_c tile.
                const int p0 = 256 * cj;
                bool released = false;
#pragma unroll 1
                for (int h = 0; h < GC / PC && g0 + PC * h < len; ++h) {
                    const int c0 = g0 + PC * h;  // first column of this pass within the tile
                    const int nbox = min(PC / 64, (len - c0) / 64);
                    if (lane == 0) bulk_wait_read0();  // previous TMA store has finished reading the staging buffer
                    __syncwarp();
#pragma unroll
                    for (int q = 0; q < PC / 64; ++q)
#pragma unroll
                        for (int c16 = 0; c16 < 8; ++c16)
                            *reinterpret_cast<uint4*>(stg + q * 4096 + lane * 128 + ((c16 ^ (lane & 7)) << 4)) =
                                make_uint4(0, 0, 0, 0);  // XOR: conflict-free 16-byte stores
                    auto put_g = [&](uint32_t w) {
                        const int j = static_cast<int>(w >> 16) - p0 - c0;
                        if (j >= 0 && j < PC)
                            *reinterpret_cast<uint16_t*>(stg + (j >> 6) * 4096 + sw128_off(lane, j & 63)) =
                                static_cast<uint16_t>(w & 0xFFFFu);
                    };
                    if (dense_blk) {
                        if (twrow) {  // TwELL tiles covering units [p0 + 128 h, p0 + 128 h + 128)
                            const int WPT = args.T / args.C, cap = WPT - 1;
                            const int t0 = (p0 + c0) / args.T, t1 = min(N, p0 + c0 + PC + args.T - 1) / args.T;
                            for (int t = t0; t < t1 && t < N / args.T; ++t) {
                                const uint32_t* blk = twrow + static_cast<int64_t>(t) * WPT;
                                const int cnt = min(static_cast<int>(__ldg(blk)), cap);
                                for (int e = 1; e <= cnt; ++e) {
                                    const uint32_t w = __ldg(blk + e);
                                    put_g(((w & 0xFFFFu) << 16) | (w >> 16));  // gate-list word: unit = position
                                }
                            }
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < UG_GPRE; ++i)
                            if (e0 + i < e1) put_g(gpre[i]);
                        for (int e = e0 + UG_GPRE; e < e1; ++e) put_g(__ldg(gl + e));
                    }
#pragma unroll 1
                    for (int q32 = 0; q32 < 2 * nbox; ++q32) {
                        uint32_t v[32];
                        tmem_ld32(tb + c0 + 32 * q32, v);
                        tmem_wait_ld();
#pragma unroll
                        for (int p = 0; p < 16; ++p) {
                            const int c = 32 * q32 + 2 * p;  // column within the half
                            uint32_t* sp = reinterpret_cast<uint32_t*>(stg + (c >> 6) * 4096 + sw128_off(lane, c & 63));
                            const uint32_t gg = *sp;
                            if (gg) {
                                const float g0 = __uint_as_float(gg << 16), g1 = __uint_as_float(gg & 0xFFFF0000u);
                                const float h0 = (gg & 0xFFFFu) ? g0 * __uint_as_float(v[2 * p]) : 0.0f;
                                const float h1 = (gg >> 16) ? g1 * __uint_as_float(v[2 * p + 1]) : 0.0f;
                                *sp = pack_bf16x2(h0, h1);
                            }
                        }
                    }
                    if (h == GC / PC - 1 || c0 + PC >= len) {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&tempty[acc]);
                        released = true;
                    }
                    fence_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        for (int q = 0; q < nbox; ++q) tma_store_2d(&tmOut, stg + q * 4096, p0 + c0 + 64 * q, row0);
                        bulk_commit();
                    }
                }
                if (!released) {  // a chunk narrower than this group's first column: nothing to store
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[acc]);
                }
            } else {
                // DOWN: rows were processed in pi order; row i of the tile goes to Y[perm[row0 + i]].
                // Stage 32 rows x 128 columns (bf16) per half in SMEM, then one 256-byte bulk copy per row.
                // DOWN: rows were processed in pi order; row i of the tile goes to Y[perm[row0 + i]].  Stage
                // 32 rows x 128 columns (bf16) per half in SMEM (conflict-free rotated 16-byte stores), then the
                // warp writes two rows per instruction with coalesced 16-byte global stores (LSU, not per-row
                // bulk copies: those were 256 small TMA requests per tile competing with the A-tile loads).
                constexpr int RB = PC * 2;            // staging bytes per row
                constexpr int LPR = RB / 16;          // lanes per row in the row writes (16 B each)
                uint32_t* srow = reinterpret_cast<uint32_t*>(stg) + lane * (RB / 4);
                const int prow_l = row0 + lane;
                const int64_t yrow_l = prow_l < args.M ? static_cast<int64_t>(__ldg(args.perm + prow_l)) : -1;
#pragma unroll 1
                for (int h = 0; h < GC / PC; ++h) {
                    const int ct = g0 + PC * h;          // column within the tile
                    const int c0 = cj * 256 + ct;        // output column
                    const int nc = min(PC, args.K - c0);
#pragma unroll 1
                    for (int ch = 0; ch < PC / 32; ++ch) {
                        uint32_t v[32];
                        tmem_ld32(tb + ct + ch * 32, v);
                        tmem_wait_ld();
                        st_row32_bf16(srow + ch * 16, v, lane);
                    }
                    if (h == GC / PC - 1) {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&tempty[acc]);
                    }
                    __syncwarp();
                    const int chunk = lane % LPR;
#pragma unroll 4
                    for (int it = 0; it < LPR; ++it) {
                        const int r = (32 / LPR) * it + lane / LPR;
                        const int64_t yrow = __shfl_sync(0xffffffffu, yrow_l, r);
                        const uint4 val = *reinterpret_cast<const uint4*>(stg + r * RB + chunk * 16);
                        if (yrow >= 0 && chunk * 8 < nc)
                            *reinterpret_cast<uint4*>(args.Y + yrow * args.K + c0 + chunk * 8) = val;
                    }
                    __syncwarp();  // staging rows read before the next pass overwrites them
                }
                if constexpr (FUSED) {
                    // this warp's 32 rows x 256 columns are in the local window: count them at the window's owner
                    // (the owner reads them through the LSA mapping, a virtual alias of the address written here)
                    asm volatile("fence.proxy.alias;" ::: "memory");
                    __threadfence_system();
                    __syncwarp();
                    if (lane == 0) {
                        const int w = b * GEMM_BM / FUSE_WIN;
                        uint32_t* f = reinterpret_cast<uint32_t*>(args.ptrs[w % args.G] + args.ptrs[args.G + 1]) + w;
                        atomicAdd_system(f, 1u);
                    }
                }
            }
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
        if (UP) {
            if (lane == 0) bulk_wait0();
        }
    }

    __syncwarp();
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem_base, 512);
    }
}

}  // namespace sffn
