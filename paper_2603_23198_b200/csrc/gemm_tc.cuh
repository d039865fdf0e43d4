// gemm_tc.cuh — persistent, warp-specialized tcgen05 GEMM for sm_100a:  D = A · B^T
//   A [M, K] bf16 row-major (K-major), B [Nout, K] bf16 row-major (K-major), fp32 accumulate in TMEM.
//
// Roles (256 threads):
//   warp 0  lane 0 : TMA producer — 128x64 A tile + 256x64 B tile per k-block into a SMEM ring
//   warp 1  lane 0 : MMA issuer   — 4 x tcgen05.mma (M=128, N=256, K=16) per k-block into one of two
//                                   TMEM accumulators (2 x 256 columns = all 512), commit -> mbarriers
//   warp 2         : TMEM allocator
//   warps 4..7     : epilogue — tcgen05.ld 32x32b (thread = output row), per-mode epilogue, TMA store
// TMEM double buffering lets the epilogue of tile i run under the mainloop of tile i+1.
//
// Epilogue modes:
//   EPI_TWELL : Alg.1 — strict > 0 on the fp32 accumulator, ascending-
//               column compaction per row and per TwELL tile of T columns, packed 32-bit words
//               (count first, idx | bf16 << 16; P:869, L1 P:817-834).  Each thread owns one row of
//               the tile, so the compaction is thread-local (no atomics, deterministic order).
//   EPI_F32   : raw fp32 accumulators (verification of the mainloop).
//   EPI_GLU   : dense baseline launch 1: B = [W_g rows n0..n0+127 ; W_u rows n0..n0+127], epilogue
//               H = bf16(relu(g) * u)  (Eq.1 P:57-60 without sparsity).
//   EPI_BF16  : dense baseline launch 2: plain bf16 store of the 128x256 tile.
#pragma once
#include "ptx.cuh"

namespace sffn {

constexpr int GEMM_BM = 128, GEMM_BN = 256, GEMM_BK = 64;
constexpr int GEMM_A_BYTES = GEMM_BM * GEMM_BK * 2;  // 16 KB
constexpr int GEMM_B_BYTES = GEMM_BN * GEMM_BK * 2;  // 32 KB
constexpr int GEMM_STAGE_BYTES = GEMM_A_BYTES + GEMM_B_BYTES;
constexpr int GEMM_THREADS = 256;
constexpr int GEMM_SMEM_LIMIT = 232448;  // max dynamic shared memory per block (227 KB)
#ifndef SFFN_GEMM_GROUP_M
#define SFFN_GEMM_GROUP_M 32
#endif
constexpr int GEMM_GROUP_M = SFFN_GEMM_GROUP_M;  // tile raster: 32 M-tiles (4096 rows) sweep all N-tiles (L2 reuse;
                                                 // 7B gate GEMM DRAM reads 3.13 -> 1.88 GB vs 16, ncu)

enum { EPI_TWELL = 0, EPI_F32 = 1, EPI_GLU = 2, EPI_BF16 = 3, EPI_BF16_MN = 4 };
// EPI_BF16_MN: as EPI_BF16, but B is given MN-major, i.e. as the [Kred, Nout] row-major matrix itself (W_d of
// the down projection, reduction over its rows): four 64-column x 64-row TMA boxes per k-block land as the
// 128B-swizzled MN-major UMMA layout (LBO 8 KB between 64-column atoms, SBO 1 KB between 8-row groups).

template <int EPI, int C>
__host__ __device__ constexpr int gemm_epi_warp_bytes() {
    return EPI == EPI_TWELL ? 32 * (GEMM_BN / C) * 4 : (EPI == EPI_F32 ? 0 : 32 * 128 * 2);  // GLU/BF16/BF16_MN
}
// Epilogue warp groups: SFFN_TWELL_EPI_GROUPS = 2 gives the TwELL epilogue (C >= 8) two groups — group g (warps
// 4+4g .. 7+4g) drains accumulator g, i.e. every other tile, two mainloops of time per tile.  Round 2 needed it at
// K = 2048 (1B) before the sparse set-bit walk: one group did not keep up (MMA thread spinning on the accumulator-free
// barrier, ncu 633k spins; tensor pipe 69%).  Other epilogues: 1 group (warps 4-7, alternating accumulators).
// Session 3: ONE group — a TwELL epilogue warp-tile takes 9.45 K cycles against a 35.5 K-cycle pair-tile mainloop at
// K = 4096 (18.5 K at K = 2048), so one group keeps up since the sparse set-bit walk; with one group and 5 ring stages
// the gate GEMM runs 0.6% (7B) / 3.9% (70B) faster (ncu, profiles/r02/s3/ncu_gate_epi.txt) and leaves 16 KB of SMEM
// and 128 threads' registers per SM free
#ifndef SFFN_TWELL_EPI_GROUPS
#define SFFN_TWELL_EPI_GROUPS 1
#endif
template <int EPI, int C>
__host__ __device__ constexpr int gemm_epi_groups() {
    return (EPI == EPI_TWELL && gemm_epi_warp_bytes<EPI, C>() <= 4096) ? SFFN_TWELL_EPI_GROUPS : 1;
}
template <int EPI, int C>
__host__ __device__ constexpr int gemm_threads() {
    return 128 + 128 * gemm_epi_groups<EPI, C>();
}
// PAIR = 2: CTA-pair (cluster of 2, cta_group::2) variant — a 256 x 256 output tile per pair, each CTA loading
// its own 128 A rows and HALF of the 256 B rows (128), the leader issuing M=256 MMAs that read both CTAs' SMEM.
// Per SM this cuts the operand stream from 48 KB to 32 KB per k-block (same MMA work).
template <int PAIR>
__host__ __device__ constexpr int gemm_stage_bytes() {
    return GEMM_A_BYTES + GEMM_B_BYTES / PAIR;
}
#ifndef SFFN_GEMM_STAGES_MAX
#define SFFN_GEMM_STAGES_MAX 6
#endif
#ifndef SFFN_TWELL_STAGES_MAX
#define SFFN_TWELL_STAGES_MAX 5  // gate GEMM ring: 5 stages measured as fast as 6 (4: +1%), session 3
#endif
template <int EPI>
__host__ __device__ constexpr int gemm_stages_max() {
    return EPI == EPI_TWELL ? SFFN_TWELL_STAGES_MAX : SFFN_GEMM_STAGES_MAX;
}
template <int EPI, int C, int PAIR = 1>
__host__ __device__ constexpr int gemm_stages() {
    return (GEMM_SMEM_LIMIT - 1024 - 256 - 4 * gemm_epi_groups<EPI, C>() * gemm_epi_warp_bytes<EPI, C>()) /
                       gemm_stage_bytes<PAIR>() > gemm_stages_max<EPI>()
               ? gemm_stages_max<EPI>()
               : (GEMM_SMEM_LIMIT - 1024 - 256 - 4 * gemm_epi_groups<EPI, C>() * gemm_epi_warp_bytes<EPI, C>()) /
                     gemm_stage_bytes<PAIR>();
}
template <int EPI, int C, int PAIR = 1>
__host__ __device__ constexpr int gemm_smem_bytes() {
    return 1024 + gemm_stages<EPI, C, PAIR>() * gemm_stage_bytes<PAIR>() +
           4 * gemm_epi_groups<EPI, C>() * gemm_epi_warp_bytes<EPI, C>() + 256;
}

struct GemmArgs {
    int M;          // rows of A / D
    int N;          // valid output columns (TwELL: hidden units; GLU: hidden units; BF16: Nout)
    int K;          // reduction length (multiple of 64 after zero fill)
    int num_m, num_n;
    int T;          // TwELL tile (EPI_TWELL)
    uint32_t* overflow;  // EPI_TWELL, may be null
    float* out_f32;      // EPI_F32
    int64_t ld_out;      // EPI_F32 row stride (elements)
    const int* m_dev;    // optional device row count: rows >= min(M, *m_dev) are skipped (dense backup rows)
    int* row_nnz;        // EPI_TWELL, may be null: += stored entries (min(count, cap)) of each row (zeroed by caller)
    int* tile_ctr;       // optional dynamic tile scheduler: tiles claimed in raster order by atomicAdd on this
                         // counter (zeroed by the caller); null: static striding (tile += grid)
    int* win_done;       // EPI_TWELL, may be null: per 2048-row window, += 1 per epilogue warp-tile whose TwELL store
                         // and row counts are complete and visible (the prep kernel, launched as a programmatic
                         // dependent, starts a window when its count reaches ceil(rows / 32) * num_n)
};
constexpr int GT_RING = 4;  // dynamic scheduler: tile ring depth (claims ahead of the slowest reader)
#ifndef SFFN_TWELL_SPARSE_MAX
#define SFFN_TWELL_SPARSE_MAX 10
#endif
constexpr int TWELL_SPARSE_MAX = SFFN_TWELL_SPARSE_MAX;  // TwELL epilogue: chunks whose rows hold <= this many positives take the sparse walk

// MN-major 128B-swizzled operand: 64-column atoms 8 KB apart (LBO), 8-row groups 1 KB apart (SBO)
__device__ __forceinline__ uint64_t umma_desc_sw128_mn_tc(uint32_t smem_addr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((smem_addr & 0x3FFFFu) >> 4);
    d |= static_cast<uint64_t>(8192 >> 4) << 16;
    d |= static_cast<uint64_t>(1024 >> 4) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(2) << 61;
    return d;
}

#ifdef SFFN_GEMM_EPI_TRACE  // probe builds only (tools/s3_epi_trace.py): cycle sums of the roles per tile
// [0] epilogue warp cycles (tfull passed -> accumulator released), [1] epilogue warp-tiles, [2] MMA cycles per tile
// (tempty passed -> last commit issued), [3] tiles, [4] MMA thread cycles waiting on tempty
static __device__ unsigned long long g_gemm_trace[8];
#endif

template <int GROUP = GEMM_GROUP_M>
__device__ __forceinline__ void gemm_tile_coords(int tile, int num_m, int num_n, int& mb, int& nb) {
    const int group = tile / (GROUP * num_n);
    const int first_m = group * GROUP;
    const int gm = min(GROUP, num_m - first_m);
    const int in = tile - group * GROUP * num_n;
    mb = first_m + in % gm;
    nb = in / gm;
}

template <int EPI, int C, int PAIR = 1>
__global__ void __launch_bounds__(gemm_threads<EPI, C>(), 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmB2, const __grid_constant__ CUtensorMap tmOut,
                   const GemmArgs args) {
    constexpr int S = gemm_stages<EPI, C, PAIR>();
    constexpr int EWB = gemm_epi_warp_bytes<EPI, C>();
    constexpr int B_BYTES = GEMM_B_BYTES / PAIR;  // this CTA's share of the B tile
    constexpr int STAGE_BYTES = gemm_stage_bytes<PAIR>();
    constexpr int PM = GEMM_BM * PAIR;            // output rows per (pair) tile
    constexpr int GROUP = GEMM_GROUP_M / PAIR;
    constexpr int NEG = gemm_epi_groups<EPI, C>();  // epilogue warp groups
    static_assert(S >= 2, "not enough shared memory for a 2-stage ring");
    static_assert(PAIR == 1 || PAIR == 2, "PAIR is 1 or 2");
    static_assert(PAIR == 1 || EPI == EPI_TWELL || EPI == EPI_F32 || EPI == EPI_BF16 || EPI == EPI_GLU,
                  "pair mode: K-major B only");

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* stA = smem;
    uint8_t* stB = smem + S * GEMM_A_BYTES;
    uint8_t* epi = stB + S * B_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(epi + 4 * NEG * EWB);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    uint64_t* tempty = tfull + 2;
    uint64_t* sfull = tempty + 2;                           // [GT_RING] dynamic tile ring: slot published
    uint64_t* sempty = sfull + GT_RING;                     // [GT_RING] slot read by every reader (leader's)
    int* sched = reinterpret_cast<int*>(sempty + GT_RING);  // [GT_RING]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sched + GT_RING);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int num_m = args.m_dev ? (min(args.M, __ldg(args.m_dev)) + PM - 1) / PM : args.num_m;
    const int num_tiles = num_m * args.num_n;
    const int nk = (args.K + GEMM_BK - 1) / GEMM_BK;
    const uint32_t rank = PAIR == 2 ? cluster_ctarank() : 0u;  // CTA rank in the pair (0 = leader / MMA issuer)
    const int first_tile = blockIdx.x / PAIR, tile_step = gridDim.x / PAIR;
    // programmatic dependent launch: once every CTA is resident, a dependent kernel (the prep kernel, which waits on
    // win_done per window instead of on this grid's completion) may be scheduled on the remaining SM resources
    if (args.win_done) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (threadIdx.x == 0) {
        tma_prefetch(&tmA);
        tma_prefetch(&tmB);
        if (EPI == EPI_GLU) tma_prefetch(&tmB2);
        if (EPI != EPI_F32) tma_prefetch(&tmOut);
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4 * PAIR);  // every epilogue warp of the pair releases the leader's accumulator
        }
        for (int i = 0; i < GT_RING; ++i) {
            mbar_init(&sfull[i], 1);
            // readers: MMA thread + the epilogue warps of every CTA (+ the peer's producer in pair mode)
            mbar_init(&sempty[i], PAIR == 2 ? 2 + 8 * NEG : 1 + 4 * NEG);
        }
        fence_mbar_init();
    }
    if (warp == 2) {
        if (PAIR == 2) tmem_alloc_pair(tmem_slot, 512);
        else tmem_alloc(tmem_slot, 512);
    }
    tc_fence_before();
    if (PAIR == 2) cluster_sync();  // peer barriers initialised before any remote arrive / complete_tx
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    // Tile sequence, identical for every role of both CTAs: static striding, or (args.tile_ctr) claims in raster
    // order by the (leader's) producer thread, published through a GT_RING-deep ring (pair: into both CTAs'
    // SMEM, st.shared::cluster + release.cluster arrive; readers release slots on the leader's sempty).  A CTA
    // (pair) that starts late takes fewer tiles, so the kernel's end is not set by its latest-starting CTA.
    const bool dyn = args.tile_ctr != nullptr;
    const uint32_t sempty_leader = PAIR == 2 ? mapa_shared(sempty, 0) : 0u;
    auto next_tile = [&](int it, int& ridx, uint32_t& rphase, bool arrive) -> int {
        if (!dyn) {
            const int t = first_tile + it * tile_step;
            return t < num_tiles ? t : -1;
        }
        if (PAIR == 2) mbar_wait_cluster(&sfull[ridx], rphase);
        else mbar_wait(&sfull[ridx], rphase);
        const int t = *reinterpret_cast<volatile int*>(&sched[ridx]);
        if (arrive) {
            if (PAIR == 2) mbar_arrive_cluster(sempty_leader + 8u * static_cast<uint32_t>(ridx));
            else mbar_arrive(&sempty[ridx]);
        }
        if (++ridx == GT_RING) {
            ridx = 0;
            rphase ^= 1;
        }
        return t;
    };

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            const uint64_t pol = policy_evict_last();
            int stage = 0;
            uint32_t phase = 0;
            int ridx = 0, widx = 0;
            uint32_t rphase = 0, wphase = 0;
            for (int it = 0;; ++it) {
                int tile;
                if (dyn && rank == 0) {  // the claiming thread
                    if (PAIR == 2) mbar_wait_cluster(&sempty[widx], wphase ^ 1);
                    else mbar_wait(&sempty[widx], wphase ^ 1);
                    tile = atomicAdd(args.tile_ctr, 1);
                    if (tile >= num_tiles) tile = -1;
                    sched[widx] = tile;
                    if (PAIR == 2) st_cluster_u32(mapa_shared(&sched[widx], 1), static_cast<uint32_t>(tile));
                    mbar_arrive(&sfull[widx]);
                    if (PAIR == 2) mbar_arrive_cluster(mapa_shared(&sfull[widx], 1));
                    if (++widx == GT_RING) {
                        widx = 0;
                        wphase ^= 1;
                    }
                } else {
                    tile = next_tile(it, ridx, rphase, true);
                }
                if (tile < 0) break;
                int mb, nb;
                gemm_tile_coords<GROUP>(tile, num_m, args.num_n, mb, nb);
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait_relaxed(&empty[stage], phase ^ 1);
                    if constexpr (PAIR == 2) {
                        // both CTAs' bytes complete on the leader's full barrier; only the leader expects them
                        const uint32_t fb = mapa_shared(&full[stage], 0);
                        if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * STAGE_BYTES);
                        tma_load_2d_pair(stA + stage * GEMM_A_BYTES, &tmA, fb, kb * GEMM_BK,
                                         mb * PM + static_cast<int>(rank) * GEMM_BM, pol);
                        if (EPI == EPI_GLU)  // B tile [W_g rows; W_u rows] of 128 hidden units: one half per CTA
                            tma_load_2d_pair(stB + stage * B_BYTES, rank == 0 ? &tmB : &tmB2, fb, kb * GEMM_BK,
                                             nb * 128, pol);
                        else
                            tma_load_2d_pair(stB + stage * B_BYTES, &tmB, fb, kb * GEMM_BK,
                                             nb * GEMM_BN + static_cast<int>(rank) * (GEMM_BN / 2), pol);
                    } else {
                    mbar_arrive_expect_tx(&full[stage], GEMM_STAGE_BYTES);
                    tma_load_2d(stA + stage * GEMM_A_BYTES, &tmA, &full[stage], kb * GEMM_BK, mb * GEMM_BM, pol);
                    if (EPI == EPI_GLU) {
                        tma_load_2d(stB + stage * GEMM_B_BYTES, &tmB, &full[stage], kb * GEMM_BK, nb * 128, pol);
                        tma_load_2d(stB + stage * GEMM_B_BYTES + GEMM_B_BYTES / 2, &tmB2, &full[stage], kb * GEMM_BK,
                                    nb * 128, pol);
                    } else if (EPI == EPI_BF16_MN) {
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            tma_load_2d(stB + stage * GEMM_B_BYTES + q * 8192, &tmB, &full[stage], nb * GEMM_BN + 64 * q,
                                        kb * GEMM_BK, pol);
                    } else {
                        tma_load_2d(stB + stage * GEMM_B_BYTES, &tmB, &full[stage], kb * GEMM_BK, nb * GEMM_BN, pol);
                    }
                    }
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer (the leader CTA in pair mode)
        if (lane == 0 && rank == 0) {
            constexpr uint32_t IDESC = umma_idesc_bf16(PM, GEMM_BN) | (EPI == EPI_BF16_MN ? (1u << 16) : 0u);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            int ridx = 0;
            uint32_t rphase = 0;
            for (int it = 0;; ++it) {
                const int tile = next_tile(it, ridx, rphase, true);
                if (tile < 0) break;
#ifdef SFFN_GEMM_EPI_TRACE
                const long long tw0 = clock64();
#endif
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
#ifdef SFFN_GEMM_EPI_TRACE
                const long long tm0 = clock64();
#endif
                const uint32_t d = tmem_base + static_cast<uint32_t>(acc * GEMM_BN);
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(stA + stage * GEMM_A_BYTES);
                    const uint32_t b0 = smem_u32(stB + stage * B_BYTES);
                    if constexpr (PAIR == 2) {
#pragma unroll
                        for (int k = 0; k < GEMM_BK / 16; ++k)
                            umma_f16_pair(d, umma_desc_sw128(a0 + k * 32), umma_desc_sw128(b0 + k * 32), IDESC,
                                          (kb | k) != 0);
                        umma_commit_pair(&empty[stage]);
                    } else {
#pragma unroll
                    for (int k = 0; k < GEMM_BK / 16; ++k)
                        umma_f16(d, umma_desc_sw128(a0 + k * 32),
                                 EPI == EPI_BF16_MN ? umma_desc_sw128_mn_tc(b0 + k * 2048) : umma_desc_sw128(b0 + k * 32),
                                 IDESC, (kb | k) != 0);
                    umma_commit(&empty[stage]);
                    }
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (PAIR == 2) umma_commit_pair(&tfull[acc]);
                else umma_commit(&tfull[acc]);
#ifdef SFFN_GEMM_EPI_TRACE
                if (EPI == EPI_TWELL) {
                    const long long tm1 = clock64();
                    atomicAdd(&g_gemm_trace[2], static_cast<unsigned long long>(tm1 - tm0));
                    atomicAdd(&g_gemm_trace[3], 1ull);
                    atomicAdd(&g_gemm_trace[4], static_cast<unsigned long long>(tm0 - tw0));
                }
#endif
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------------------------ epilogue
        const int ew = (warp - 4) & 3;   // TMEM lane quarter accessible to this warp (warp % 4)
        const int eg = (warp - 4) >> 2;  // epilogue group: with NEG == 2, group g drains accumulator g
        uint8_t* stg = epi + (warp - 4) * EWB;
        int acc = NEG == 2 ? eg : 0;
        uint32_t acc_phase = 0;
        const uint32_t tempty_leader = PAIR == 2 ? mapa_shared(tempty, 0) : 0u;
        auto release_acc = [&](int a) {  // lane 0: this warp is done reading accumulator a
            if (PAIR == 2) mbar_arrive_remote(tempty_leader + 8u * static_cast<uint32_t>(a));
            else mbar_arrive(&tempty[a]);
        };
        int ridx = 0;
        uint32_t rphase = 0;
        for (int it = 0;; ++it) {
            const int tile = next_tile(it, ridx, rphase, lane == 0);
            if (tile < 0) break;
            if (NEG == 2 && (it & 1) != eg) continue;  // the other group's tile (accumulator)
            int mb, nb;
            gemm_tile_coords<GROUP>(tile, num_m, args.num_n, mb, nb);
            const int row0 = mb * PM + static_cast<int>(rank) * GEMM_BM + ew * 32;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
#ifdef SFFN_GEMM_EPI_TRACE
            const long long te0 = clock64();
#endif
            const uint32_t tb = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + static_cast<uint32_t>(acc * GEMM_BN);
            if (EPI != EPI_F32) {
                if (lane == 0) bulk_wait_read0();  // staging buffer free (previous TMA store has read it)
                __syncwarp();
            }
            if constexpr (EPI == EPI_TWELL) {
                constexpr int ROW_WORDS = GEMM_BN / C;
                // staging of the warp's 32 rows x ROW_WORDS packed words: for C <= 8 as ROW_WORDS/32 boxes of
                // 32 rows x 128 B in the TMA 128-byte-swizzle layout (16-byte chunk index XOR row % 8), so the 32
                // lanes (= 32 rows) writing the same word index hit 8 different bank groups instead of one bank;
                // C = 16 (64-byte rows): plain row-major
                constexpr bool SWZ = ROW_WORDS % 32 == 0;
                const int T = args.T;
                const int WPT = T / C;
                const int cap = WPT - 1;
                uint8_t* sbase = stg;
                auto sword = [&](int p) -> uint32_t* {
                    if constexpr (SWZ)
                        return reinterpret_cast<uint32_t*>(sbase + (p >> 5) * 4096 + lane * 128 +
                                                           ((((p >> 2) & 7) ^ (lane & 7)) << 4) + ((p & 3) << 2));
                    else
                        return reinterpret_cast<uint32_t*>(sbase) + lane * ROW_WORDS + p;
                };
                const int col_base = nb * GEMM_BN;
                const bool row_ok = row0 + lane < args.M;
                int z = 0, stored = 0;
#pragma unroll 1
                for (int ch = 0; ch < GEMM_BN / 32; ++ch) {
                    uint32_t v[32];
                    tmem_ld32(tb + ch * 32, v);
                    tmem_wait_ld();
                    const int tcol = ch * 32;
                    if (tcol % T == 0) z = 0;
                    const int tbase = (tcol / T) * WPT;  // word of this tile's count within the row
                    // Alg.1 line 11 (strict > 0 on the fp32 accumulator) as a 32-bit mask of the chunk's columns;
                    // lines 12-15 as mask/popc compaction: the slot of column i is the running count z plus the
                    // positives before it, popc(mask & (2^i - 1)) — ascending column order, no atomics, and the
                    // (usual, at 99% sparsity) all-zero chunk costs only the compares
                    uint32_t mask = 0;
#pragma unroll
                    for (int i = 0; i < 32; ++i) mask |= (__uint_as_float(v[i]) > 0.0f ? 1u : 0u) << i;
#ifdef SFFN_TWELL_PROBE_NOEPI  // timing probe (tools): the compaction skipped, results wrong
                    if (mask != 0x12345678u) { z += __popc(mask); continue; }
#endif
                    // columns positive in ANY of the warp's 32 rows (~10 of 32 at 1% density): a warp-uniform
                    // branch per column skips the rest, so the compaction costs ~ the positives, not 32 columns
                    // (at K = 2048 the epilogue, not the mainloop, bounded the kernel: tensor pipe 69%, ncu 1B)
                    // Sparse chunks (at most TWELL_SPARSE_MAX = 10 positives in every row; A/B of 3 / 6 / 10: 10 best at 95% and 99%): walk the row's own set
                    // bits — a warp-uniform trip count = the most positives any lane has — and pick each value with a
                    // 5-level select tree over the 32 registers (no dynamic register indexing), so a chunk costs ~the
                    // positives instead of 32 columns of slot arithmetic.  The k-th positive goes to slot z + k.
                    const int wmax = __reduce_max_sync(0xffffffffu, static_cast<uint32_t>(__popc(mask)));
                    if (wmax <= TWELL_SPARSE_MAX) {
                        uint32_t m = mask;
                        for (int k = 0; k < wmax; ++k) {
                            if (m) {
                                const int i = __ffs(m) - 1;
                                m &= m - 1;
                                const int slot = z + k;
                                if (slot < cap) {
                                    uint32_t a16[16], a8[8], a4[4], a2[2];
#pragma unroll
                                    for (int j = 0; j < 16; ++j) a16[j] = (i & 16) ? v[j + 16] : v[j];
#pragma unroll
                                    for (int j = 0; j < 8; ++j) a8[j] = (i & 8) ? a16[j + 8] : a16[j];
#pragma unroll
                                    for (int j = 0; j < 4; ++j) a4[j] = (i & 4) ? a8[j + 4] : a8[j];
#pragma unroll
                                    for (int j = 0; j < 2; ++j) a2[j] = (i & 2) ? a4[j + 2] : a4[j];
                                    const uint32_t x = (i & 1) ? a2[1] : a2[0];
                                    const uint32_t bf = __bfloat16_as_ushort(__float2bfloat16_rn(__uint_as_float(x)));
                                    *sword(tbase + 1 + slot) = static_cast<uint32_t>(col_base + tcol + i) | (bf << 16);
                                }
                            }
                        }
                    } else if (mask) {
                        // dense chunks: every column's store predicated on its bit (no per-column branch; the former
                        // warp-uniform branch per column cost a BSSY/BSYNC reconvergence each)
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            const int slot = z + __popc(mask & ((1u << i) - 1u));
                            const bool st = ((mask >> i) & 1u) && slot < cap;
                            const uint32_t bf = __bfloat16_as_ushort(__float2bfloat16_rn(__uint_as_float(v[i])));
                            uint32_t* dst = sword(tbase + 1 + slot);
                            const uint32_t w = static_cast<uint32_t>(col_base + tcol + i) | (bf << 16);
                            asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.shared.u32 [%0], %1;\n\t}"
                                         ::"r"(smem_u32(dst)), "r"(w), "r"(static_cast<uint32_t>(st)) : "memory");
                        }
                    }
                    z += __popc(mask);
                    if ((tcol + 32) % T == 0) {
                        *sword(tbase) = static_cast<uint32_t>(z);  // Alg.1 line 17: true count
                        if (z > cap && row_ok && args.overflow) atomicAdd(args.overflow, 1u);
                        stored += min(z, cap);
                    }
                }
                if (args.row_nnz && row_ok && stored) atomicAdd(args.row_nnz + row0 + lane, stored);
                if (args.win_done) __threadfence();  // the row counts before the window signal below
                tc_fence_before();
                __syncwarp();
                if (lane == 0) release_acc(acc);
#ifdef SFFN_GEMM_EPI_TRACE
                if (lane == 0) {
                    atomicAdd(&g_gemm_trace[0], static_cast<unsigned long long>(clock64() - te0));
                    atomicAdd(&g_gemm_trace[1], 1ull);
                }
#endif
                fence_async_smem();
                __syncwarp();
                if (lane == 0) {
                    // TwELL is a streaming output: L2 evict_first keeps X / W_g resident (gate GEMM -0.3%, ncu A/B)
                    if constexpr (SWZ) {
#pragma unroll
                        for (int q = 0; q < ROW_WORDS / 32; ++q)
                            tma_store_2d_hint(&tmOut, stg + q * 4096, nb * ROW_WORDS + 32 * q, row0, policy_evict_first());
                    } else {
                        tma_store_2d_hint(&tmOut, stg, nb * ROW_WORDS, row0, policy_evict_first());
                    }
                    bulk_commit();
                    if (args.win_done && row0 < args.M) {
                        // the store complete (writes performed), ordered before the generic-proxy signal, released
                        bulk_wait0();
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                        __threadfence();
                        atomicAdd(args.win_done + (row0 >> 11), 1);
                    }
                }
            } else if constexpr (EPI == EPI_F32) {
                const int row = row0 + lane;
#pragma unroll 1
                for (int ch = 0; ch < GEMM_BN / 32; ++ch) {
                    uint32_t v[32];
                    tmem_ld32(tb + ch * 32, v);
                    tmem_wait_ld();
                    const int col = nb * GEMM_BN + ch * 32;
                    if (row < args.M) {
                        float* o = args.out_f32 + static_cast<int64_t>(row) * args.ld_out + col;
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            if (col + 4 * j < args.N)
                                *reinterpret_cast<uint4*>(o + 4 * j) = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) release_acc(acc);
            } else if constexpr (EPI == EPI_GLU) {
                uint32_t* srow = reinterpret_cast<uint32_t*>(stg) + lane * 64;  // 128 bf16 per row
#pragma unroll 1
                for (int ch = 0; ch < 4; ++ch) {
                    uint32_t g[32], u[32];
                    tmem_ld32(tb + ch * 32, g);
                    tmem_ld32(tb + 128 + ch * 32, u);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        g[j] = __float_as_uint(fmaxf(__uint_as_float(g[j]), 0.0f) * __uint_as_float(u[j]));
                    st_row32_bf16(srow + ch * 16, g, lane);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) release_acc(acc);
                fence_async_smem();
                __syncwarp();
                if (lane == 0) {
                    tma_store_2d(&tmOut, stg, nb * 128, row0);
                    bulk_commit();
                }
            } else {  // EPI_BF16, EPI_BF16_MN
                uint32_t* srow = reinterpret_cast<uint32_t*>(stg) + lane * 64;
#pragma unroll 1
                for (int half = 0; half < 2; ++half) {
                    if (half == 1) {
                        if (lane == 0) bulk_wait_read0();
                        __syncwarp();
                    }
#pragma unroll 1
                    for (int ch = 0; ch < 4; ++ch) {
                        uint32_t v[32];
                        tmem_ld32(tb + half * 128 + ch * 32, v);
                        tmem_wait_ld();
                        st_row32_bf16(srow + ch * 16, v, lane);
                    }
                    if (half == 1) {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) release_acc(acc);
                    }
                    fence_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        tma_store_2d(&tmOut, stg, nb * GEMM_BN + half * 128, row0);
                        bulk_commit();
                    }
                }
            }
            if (NEG == 2) {
                acc_phase ^= 1;
            } else if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
        if (lane == 0) bulk_wait0();
    }

    __syncwarp();
    tc_fence_before();
    if (PAIR == 2) cluster_sync();  // the leader's MMAs write the peer's TMEM; remote arrives target the leader
    else __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        if (PAIR == 2) tmem_dealloc_pair(tmem_base, 512);
        else tmem_dealloc(tmem_base, 512);
    }
}

}  // namespace sffn
