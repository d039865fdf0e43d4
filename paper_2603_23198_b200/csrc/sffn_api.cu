// sffn_api.cu — host side of the C ABI declared in include/sffn.h: argument validation, TMA tensor-map
// encoding (cuTensorMapEncodeTiled via the runtime's driver entry point, no -lcuda), launches.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/sffn.h"
#include "gemm_tc.cuh"
#include "fp32_path.cuh"
#include "gemm_union.cuh"
#include "gemm_union_pair.cuh"
#include "prep.cuh"
#include "hybrid.cuh"
#include "hybrid_mm.cuh"
#include "updown.cuh"

using namespace sffn;

// host-side count of the kernels this library has launched (or captured into a graph): sffn_launch_count()
static std::atomic<long long> g_launches{0};
static inline void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

namespace {

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                       const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                       CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled_t encode_fn() {
    static PFN_encodeTiled_t fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_encodeTiled_t>(p);
    }();
    return fn;
}

// 2-D row-major tensor [outer, inner] of `esize`-byte elements, box [box_outer, box_inner].
bool tmap_2d(CUtensorMap* m, CUtensorMapDataType dt, int esize, const void* ptr, uint64_t inner, uint64_t outer,
             uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle sw) {
    PFN_encodeTiled_t enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {inner * static_cast<uint64_t>(esize)};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

struct DevInfo {
    int sms = 0;
    int major = 0;
};
DevInfo dev_info() {
    int dev = 0;
    DevInfo d;
    if (cudaGetDevice(&dev) != cudaSuccess) return d;
    cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&d.major, cudaDevAttrComputeCapabilityMajor, dev);
    return d;
}

// tuning override for raster group sizes (unset in production: the compiled defaults apply)
int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    if (!v || !*v) return dflt;
    const int x = std::atoi(v);
    return x > 0 ? x : dflt;
}

// on/off switch for A/B comparisons: "0" disables, anything else (or unset) keeps the default
bool env_flag(const char* name, bool dflt) {
    const char* v = std::getenv(name);
    if (!v || !*v) return dflt;
    return std::atoi(v) != 0;
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

bool valid_TC(int T, int C) {
    if (!(T == 32 || T == 64 || T == 128 || T == 256)) return false;
    if (!(C == 1 || C == 2 || C == 4 || C == 8 || C == 16)) return false;
    return T / C >= 2;
}

// PAIR = 2 launches clusters of two CTAs (one CTA pair per TPC, cta_group::2 MMAs); the B tensor map must then
// have a 128-row box (each CTA loads half of the 256-row B tile).
template <int EPI, int C, int PAIR = 1>
int launch_gemm(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& b2, const CUtensorMap& o,
                GemmArgs args, int n_tile_cols, cudaStream_t st) {
    auto kern = gemm_tc_kernel<EPI, C, PAIR>;
    constexpr int smem = gemm_smem_bytes<EPI, C, PAIR>();
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [&] {
        attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (attr_err == cudaSuccess)  // the same carveout as the overlapped prep kernel (co-residency)
            attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                            cudaSharedmemCarveoutMaxShared);
    });
    if (attr_err != cudaSuccess) return SFFN_ERR_CUDA;
    args.num_m = (args.M + GEMM_BM * PAIR - 1) / (GEMM_BM * PAIR);
    args.num_n = (args.N + n_tile_cols - 1) / n_tile_cols;
    const int tiles = args.num_m * args.num_n;
    if (tiles == 0) return SFFN_OK;
    DevInfo d = dev_info();
    if constexpr (PAIR == 1) {
        const int grid = tiles < d.sms ? tiles : d.sms;
        { kern<<<grid, gemm_threads<EPI, C>(), smem, st>>>(a, b, b2, o, args); note_launch(); }
    } else {
        const int pairs = tiles < d.sms / 2 ? tiles : d.sms / 2;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(2 * pairs);
        cfg.blockDim = dim3(gemm_threads<EPI, C>());
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        if (cudaLaunchKernelEx(&cfg, kern, a, b, b2, o, args) != cudaSuccess) return SFFN_ERR_CUDA;
        note_launch();
    }
    return cudaGetLastError() == cudaSuccess ? SFFN_OK : SFFN_ERR_CUDA;
}

int check_device() {
    DevInfo d = dev_info();
    if (d.sms == 0) return SFFN_ERR_CUDA;
    if (d.major != 10) return SFFN_ERR_UNSUPPORTED;
    return SFFN_OK;
}

int pack_impl(const void* X, const void* Wg, int64_t M, int64_t K, int64_t N, int T, int C, uint32_t* twell,
              uint32_t* d_overflow, cudaStream_t st, int* row_nnz = nullptr, int* tile_ctr = nullptr,
              int* win_done = nullptr) {
    // CTA-pair gate GEMM by default (SFFN_GATE_PAIR=0 selects the single-CTA kernel)
    static const bool pair = env_flag("SFFN_GATE_PAIR", true);
    CUtensorMap ta, tb, to;
    if (!tmap_2d(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, X, K, M, GEMM_BK, GEMM_BM, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !tmap_2d(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Wg, K, N, GEMM_BK, pair ? GEMM_BN / 2 : GEMM_BN,
                 CU_TENSOR_MAP_SWIZZLE_128B) ||
        // TwELL store boxes: 32 rows x 32 words, 128-byte swizzled, for C <= 8 (gemm_tc.cuh EPI_TWELL staging);
        // 32 rows x 16 words unswizzled for C = 16
        !tmap_2d(&to, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, twell, N / C, M, C <= 8 ? 32 : GEMM_BN / C, 32,
                 C <= 8 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE))
        return SFFN_ERR_CUDA;
    GemmArgs args{};
    args.M = static_cast<int>(M);
    args.N = static_cast<int>(N);
    args.K = static_cast<int>(K);
    args.T = T;
    args.overflow = d_overflow;
    args.row_nnz = row_nnz;
    args.tile_ctr = env_flag("SFFN_GATE_DYN", false) ? tile_ctr : nullptr;  // measured neutral: off
    args.win_done = win_done;
#define SFFN_PACK_CASE(CC)                                                                              \
    case CC:                                                                                            \
        return pair ? launch_gemm<EPI_TWELL, CC, 2>(ta, tb, tb, to, args, GEMM_BN, st)                  \
                    : launch_gemm<EPI_TWELL, CC, 1>(ta, tb, tb, to, args, GEMM_BN, st);
    switch (C) {
        SFFN_PACK_CASE(1)
        SFFN_PACK_CASE(2)
        SFFN_PACK_CASE(4)
        SFFN_PACK_CASE(8)
        SFFN_PACK_CASE(16)
    }
#undef SFFN_PACK_CASE
    return SFFN_ERR_INVALID_ARG;
}

int pack_checks(const void* X, const void* Wg, int64_t M, int64_t K, int64_t N, int T, int C, const void* out) {
    if (M == 0 && valid_TC(T, C)) X = out = Wg;  // empty batch: X / out may be NULL (nothing is touched)
    if (!X || !Wg || !out) return SFFN_ERR_INVALID_ARG;
    if (!aligned16(X) || !aligned16(Wg) || !aligned16(out)) return SFFN_ERR_INVALID_ARG;
    if (!valid_TC(T, C)) return SFFN_ERR_INVALID_ARG;
    if (M < 0 || K < 64 || K % 64 != 0 || N <= 0 || N % T != 0 || N % 16 != 0 || N > 65536) return SFFN_ERR_SHAPE;
    if (M > (int64_t(1) << 31) - GEMM_BM || K > (int64_t(1) << 30)) return SFFN_ERR_SHAPE;
    return SFFN_OK;
}

int updown_impl(const void* X, const uint32_t* tw, const void* Wu, const void* Wd, int64_t M, int64_t K, int64_t N,
                int T, int C, void* Y, cudaStream_t st) {
    if (M == 0) return SFFN_OK;
    const int64_t K8 = K / 8;
    const int64_t per_warp = (K8 + UD_WARPS - 1) / UD_WARPS;  // chunks per warp
    const int nch_needed = static_cast<int>((per_warp + 31) / 32);
    dim3 grid(static_cast<unsigned>(M)), block(UD_WARPS * 32);
    const uint4* x = static_cast<const uint4*>(X);
    const uint4* wu = static_cast<const uint4*>(Wu);
    const uint4* wd = static_cast<const uint4*>(Wd);
    uint4* y = static_cast<uint4*>(Y);
    if (nch_needed <= 1)
        { updown_kernel<1><<<grid, block, 0, st>>>(x, tw, wu, wd, y, (int)M, (int)K, (int)N, T, C); note_launch(); }
    else if (nch_needed <= 2)
        { updown_kernel<2><<<grid, block, 0, st>>>(x, tw, wu, wd, y, (int)M, (int)K, (int)N, T, C); note_launch(); }
    else if (nch_needed <= 4)
        { updown_kernel<4><<<grid, block, 0, st>>>(x, tw, wu, wd, y, (int)M, (int)K, (int)N, T, C); note_launch(); }
    else if (nch_needed <= 8)
        { updown_kernel<8><<<grid, block, 0, st>>>(x, tw, wu, wd, y, (int)M, (int)K, (int)N, T, C); note_launch(); }
    else
        return SFFN_ERR_SHAPE;
    return cudaGetLastError() == cudaSuccess ? SFFN_OK : SFFN_ERR_CUDA;
}

int resolve_algo(int algo, int64_t N);

// argument / shape checks of the up/down entry points; the GATHER kernel keeps x in registers (K <= 8192), the
// UNION tensor-core path tiles K (K <= 65536)
int updown_checks(const void* X, const void* tw, const void* Wu, const void* Wd, int64_t M, int64_t K, int64_t N,
                  int T, int C, const void* Y, int algo) {
    if (M == 0) X = tw = Y = Wu;  // empty batch: X / twell / Y may be NULL
    if (!X || !tw || !Wu || !Wd || !Y) return SFFN_ERR_INVALID_ARG;
    if (!aligned16(X) || !aligned16(tw) || !aligned16(Wu) || !aligned16(Wd) || !aligned16(Y))
        return SFFN_ERR_INVALID_ARG;
    if (!valid_TC(T, C)) return SFFN_ERR_INVALID_ARG;
    if (M < 0 || K < 64 || K % 64 != 0 || K > 65536 || N <= 0 || N % T != 0 || N > 65536) return SFFN_ERR_SHAPE;
    if (K > 8192 && N > 0 && resolve_algo(algo, N) == SFFN_ALGO_GATHER) return SFFN_ERR_SHAPE;
    if (M > 2147483647) return SFFN_ERR_SHAPE;
    return SFFN_OK;
}


// ---------------------------------------------------------------- block-union tensor-core up/down
inline int64_t align1k(int64_t x) { return (x + 1023) & ~int64_t(1023); }

struct UnionWs {
    int64_t hc, ulist, ulen, utot, udense, umask, uwoff, chunk, tiles, perm, xp, ctr, nnz, pctr, glist, coff, total;
    int lmax, nchunk;
};
// Token rows per union block: 128 (single-CTA union GEMMs) or 256 (CTA-pair union GEMMs, SFFN_UNION_PAIR=1).
int union_brows() {
    static const int br = env_flag("SFFN_UNION_PAIR", false) ? 256 : 128;
    return br;
}

UnionWs union_ws_layout(int64_t M, int64_t N, int64_t K, int T = 256, int C = 8) {
    const int64_t BR = union_brows();
    const int64_t NB = (M + BR - 1) / BR;
    UnionWs w{};
    int64_t o = 0;
    w.hc = o;    o = align1k(o + NB * BR * N * 2);
    w.ulist = o; o = align1k(o + NB * N * 4);
    w.ulen = o;  o = align1k(o + NB * 4);
    w.utot = o;  o = align1k(o + NB * 4);
    w.udense = o; o = align1k(o + NB * 4);
    w.uwoff = o; o = align1k(o + NB * (N / 32) * 4);
    w.chunk = o; o = align1k(o + (NB + 1) * 4);
    w.tiles = o; o = align1k(o + NB * ((N + 255) / 256) * 4);
    w.perm = o;  o = align1k(o + M * 4);
    w.xp = o;    o = align1k(o + M * K * 2);
    w.ctr = o;   o = align1k(o + 64);
    // zeroed together before each forward (one memset): row counts + the gate GEMM's tile counter (nnz[M]), the
    // prep kernel's counters, and (split prep only) the merged union masks
    w.nnz = o;   o = (o + (M + 1) * 4 + 15) & ~int64_t(15);
    w.pctr = o;  o = (o + (2 + 2 * NB + (M + 2047) / 2048) * 4 + 15) & ~int64_t(15);  // + gate->prep window counters
    w.umask = o; o = align1k(o + NB * (N / 32) * 4);
    w.lmax = static_cast<int>((N / T) * (T / C - 1));  // most stored entries a row can have
    w.nchunk = static_cast<int>((N + 255) / 256);
    w.glist = o; o = align1k(o + NB * BR * static_cast<int64_t>(w.lmax) * 4);
    w.coff = o;  o = align1k(o + NB * BR * static_cast<int64_t>(w.nchunk + 1) * 2);
    w.total = o;
    return w;
}

bool union_applicable(int64_t N) { return N % 64 == 0 && N >= 64; }

int resolve_algo(int algo, int64_t N) {
    if (algo == SFFN_ALGO_AUTO) return union_applicable(N) ? SFFN_ALGO_UNION : SFFN_ALGO_GATHER;
    return algo;
}

size_t updown_ws_bytes(int64_t M, int64_t N, int64_t K, int algo, int T = 32, int C = 1) {
    // sized for the worst (T, C) unless given: the gate lists need (N/T)*(T/C-1) entries per row
    if (resolve_algo(algo, N) != SFFN_ALGO_UNION || M <= 0) return 0;
    return static_cast<size_t>(union_ws_layout(M, N, K, T, C).total);
}

// Row nnz buffer of the union workspace (sffn_forward lets the gate GEMM epilogue fill it: nnz_ready)
int* union_nnz_ptr(void* ws, int64_t M, int64_t N, int64_t K, int T, int C) {
    return reinterpret_cast<int*>(static_cast<uint8_t*>(ws) + union_ws_layout(M, N, K, T, C).nnz);
}

// tools: per-CTA phase timestamps of the prep kernel (SFFN_PREP_TRACE=1; sffn__prep_trace copies them out)
unsigned long long* g_prep_trace = nullptr;
int64_t g_prep_trace_n = 0;
unsigned long long* prep_trace_buf(int64_t ctas) {
    static const bool on = env_flag("SFFN_PREP_TRACE", false);
    if (!on) return nullptr;
    if (ctas * 8 > g_prep_trace_n) {
        if (g_prep_trace) cudaFree(g_prep_trace);
        if (cudaMalloc(&g_prep_trace, static_cast<size_t>(ctas) * 64) != cudaSuccess) return nullptr;
        g_prep_trace_n = ctas * 8;
    }
    cudaMemset(g_prep_trace, 0, static_cast<size_t>(g_prep_trace_n) * 8);
    return g_prep_trace;
}

// CTAs per union block of the prep kernel: a power of two (it must divide the block rows), up to ~1.5 waves of CTAs
// densest-blocks-first split of the prep kernel (prep_parts): the strongest boost whose CTAs fit in one wave of 2 CTAs
// per SM; SFFN_PREP_BOOST=0/1/2 forces one (A/B)
int union_prep_split(int64_t NB);
int union_prep_boost(int64_t NB, int BR) {
    const char* e = std::getenv("SFFN_PREP_BOOST");
    if (e && *e) return std::min(2, std::max(0, std::atoi(e)));
    const int base = union_prep_split(NB), sms = dev_info().sms;
    for (int b = 2; b > 0; --b)
        if (prep_ctas(static_cast<int>(NB), PERM_W / BR, base, b) <= 2 * sms) return b;
    return 0;
}

int union_prep_split(int64_t NB) {
    const int forced = env_int("SFFN_PREP_SPLIT", 0);  // tuning override (power of two <= META_SPLIT_MAX)
    if (forced > 0 && forced <= META_SPLIT_MAX && (forced & (forced - 1)) == 0) return forced;
    const int sms = dev_info().sms;
    int split = 1;
    while (split < META_SPLIT_MAX && 2 * NB * split < 3 * sms) split *= 2;
    return split;
}

// Overlapped prep (session 3): the gate GEMM signals per 2048-row window (GemmArgs::win_done) and starts the prep
// kernel as a programmatic dependent; prep CTAs run beside the gate GEMM (one per SM: 256 + 512 threads, 28.7 K + 32 K
// registers, 181 KB + the prep's SMEM) and wait per window.  SFFN_PREP_OVERLAP=0/1 (A/B; default below).
#ifndef SFFN_PREP_OVERLAP_DEFAULT
#define SFFN_PREP_OVERLAP_DEFAULT 0
#endif
bool union_prep_overlap_enabled() { return env_flag("SFFN_PREP_OVERLAP", SFFN_PREP_OVERLAP_DEFAULT != 0); }
constexpr int PREP_TAIL_SPLIT = 8;  // parts per block of the windows the gate GEMM finishes last
// X-copy ring piece that lets a prep CTA sit beside a gate GEMM CTA (0: does not fit -> no overlap)
int prep_overlap_piece(int64_t N, int nchunk, int C) {
    int gsmem = 0;
    switch (C) {
        case 1: gsmem = gemm_smem_bytes<EPI_TWELL, 1, 2>(); break;
        case 2: gsmem = gemm_smem_bytes<EPI_TWELL, 2, 2>(); break;
        case 4: gsmem = gemm_smem_bytes<EPI_TWELL, 4, 2>(); break;
        case 8: gsmem = gemm_smem_bytes<EPI_TWELL, 8, 2>(); break;
        default: gsmem = gemm_smem_bytes<EPI_TWELL, 16, 2>(); break;
    }
    const int64_t budget = 233472 - 2 * 1024 - gsmem - PREP_STATIC_SMEM;  // 228 KB per SM, 1 KB reserved per CTA
    for (int piece : {8192, 6144, 4096, 3072, 2048})
        if (static_cast<int64_t>(prep_smem_bytes(static_cast<int>(N), nchunk, piece)) <= budget) return piece;
    return 0;
}
// the gate GEMM's last raster group (GEMM_GROUP_M / 2 pair-M-tiles) -> first window it covers
int prep_tail_w0(int64_t M) {
    const int64_t pm = (M + 255) / 256, grp = GEMM_GROUP_M / 2;
    return static_cast<int>(((pm - 1) / grp) * grp * 256 / 2048);
}

// Bytes to zero before a gated union forward, from the row-count buffer (union_nnz_ptr) on: row counts, the gate
// GEMM tile counter, the prep kernel's counters and, when the prep kernel splits blocks, the merged masks.
size_t union_zero_bytes(int64_t M, int64_t N, int64_t K, int T, int C) {
    const UnionWs L = union_ws_layout(M, N, K, T, C);
    const int64_t NB = (M + union_brows() - 1) / union_brows();
    const int64_t end = (union_prep_split(NB) > 1 || union_prep_boost(NB, union_brows()) || union_prep_overlap_enabled())
                            ? L.umask + NB * (N / 32) * 4
                            : L.pctr + (2 + 2 * NB + (M + 2047) / 2048) * 4;
    return static_cast<size_t>(end - L.nnz);
}

// Union size from which a block is made dense (all N units; its weight tiles then come by TMA instead of
// gathers): SFFN_UNION_DENSE (fraction of N, default 0.7; >= 1 disables).  Only the single-CTA kernels have the
// TMA path (and it needs N >= 256 for the UP box); the pair kernels would keep gathering an identity list.
int union_dense_units(int64_t N, bool has_tma_path) {
    static const double frac = [] {
        const char* e = std::getenv("SFFN_UNION_DENSE");
        return e ? std::atof(e) : 0.7;
    }();
    if (!has_tma_path || frac >= 1.0) return static_cast<int>(N) + 1;
    return std::max(1, static_cast<int>(frac * static_cast<double>(N)));
}

// Stored entries of a block (summed over its rows) from which the block is made dense without computing its
// union: SFFN_UNION_DENSE_NNZ (multiple of N, default 8; 0 disables).  At 99% sparsity a 128-row block holds
// ~1.3 N entries on average and up to ~4.5 N in the densest blocks (union <= 0.66 N: with a threshold of 4 those
// went dense and the 7B union GEMMs lost 9%); at 95% ~6.4 N, at 90% ~13 N (union ~N).
int64_t union_dense_nnz(int64_t N, bool has_tma_path) {
    static const double f = [] {
        const char* e = std::getenv("SFFN_UNION_DENSE_NNZ");
        return e ? std::atof(e) : 8.0;
    }();
    if (!has_tma_path || f <= 0.0) return INT64_MAX;
    return static_cast<int64_t>(f * static_cast<double>(N));
}

// NEXT-3 fused all-reduce parameters of the DOWN kernel (sffn_sharded_forward_fused; null: plain DOWN)
struct FuseParams {
    const uint64_t* ptrs;  // device: G window bases, multicast base (0 if none), counter-set offset
    int G, rank;
    int phase;  // 0: the whole up/down; 1: everything before the DOWN kernel; 2: the DOWN kernel only
};

// ov_piece > 0: the gate GEMM was launched with win_done = the prep counters' window block (union_win_done) and the
// prep kernel is launched as its programmatic dependent with an X-copy ring of 8 x ov_piece bytes (prep_overlap_piece)
int union_updown_impl(const void* X, const uint32_t* tw, const void* Wu, const void* Wd, int64_t M, int64_t K,
                      int64_t N, int T, int C, void* Y, void* ws, cudaStream_t st, bool gated = true,
                      bool nnz_ready = false, const FuseParams* fuse = nullptr, int ov_piece = 0) {
    const int BR = union_brows();
    const int64_t NB = (M + BR - 1) / BR;
    UnionWs L = union_ws_layout(M, N, K, T, C);
    uint8_t* base = static_cast<uint8_t*>(ws);
    UnionMeta um;
    um.ulist = reinterpret_cast<int32_t*>(base + L.ulist);
    um.ulen = reinterpret_cast<int32_t*>(base + L.ulen);
    um.utot = reinterpret_cast<int32_t*>(base + L.utot);
    um.udense = reinterpret_cast<int32_t*>(base + L.udense);
    um.umask = reinterpret_cast<uint32_t*>(base + L.umask);
    um.uwoff = reinterpret_cast<int32_t*>(base + L.uwoff);
    um.chunk_off = reinterpret_cast<int32_t*>(base + L.chunk);
    um.tiles = reinterpret_cast<int32_t*>(base + L.tiles);
    um.counters = reinterpret_cast<int*>(base + L.ctr);
    um.glist = reinterpret_cast<uint32_t*>(base + L.glist);
    um.coff = reinterpret_cast<uint16_t*>(base + L.coff);
    um.lmax = L.lmax;
    um.nchunk = L.nchunk;
    um.brows = BR;
    void* hc = base + L.hc;
    int32_t* perm = reinterpret_cast<int32_t*>(base + L.perm);
    void* xp = base + L.xp;
    // row permutation pi (per 2048-row window, descending stored nnz) and the permuted copy of X
    int* rnnz = reinterpret_cast<int*>(base + L.nnz);
    const int phase = fuse ? fuse->phase : 0;
    if (phase != 2) {
        // one prep launch: pi, unions, work list, gate lists and X in pi order (prep.cuh); the non-gated variant needs
        // neither gate lists nor X and scatters the TwELL values into H_c instead (no UP GEMM)
        if (!nnz_ready) {
            { row_nnz_kernel<<<static_cast<unsigned>((M * 32 + 255) / 256), 256, 0, st>>>(tw, (int)M, (int)N, T, C, rnnz); note_launch(); }
            if (cudaGetLastError() != cudaSuccess) return SFFN_ERR_CUDA;
            if (cudaMemsetAsync(base + L.pctr, 0, union_zero_bytes(M, N, K, T, C) - static_cast<size_t>(L.pctr - L.nnz),
                                st) != cudaSuccess)
                return SFFN_ERR_CUDA;
        }
        const bool ovl = ov_piece > 0;
        const int split = union_prep_split(NB), boost = ovl ? 1 : union_prep_boost(NB, BR);
        PrepOv ov{};
        int pctas;
        if (ovl) {
            ov.win_done = reinterpret_cast<const int*>(base + L.pctr) + 2 + 2 * NB;
            ov.win_n = static_cast<int>((N + GEMM_BN - 1) / GEMM_BN);
            ov.tail_w0 = prep_tail_w0(M);
            ov.tail_split = std::max(split, PREP_TAIL_SPLIT);
            pctas = prep_ctas_ov(static_cast<int>(NB), PERM_W / BR, split, boost, ov.tail_w0, ov.tail_split);
        } else {
            pctas = prep_ctas(static_cast<int>(NB), PERM_W / BR, split, boost);
        }
        const int piece = ovl ? ov_piece : PREP_PIECE;
        const size_t psmem = prep_smem_bytes(static_cast<int>(N), L.nchunk, piece);
        static std::once_flag ponce;
        static cudaError_t pattr = cudaSuccess;
        std::call_once(ponce, [] {
            pattr = cudaFuncSetAttribute(union_prep_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(prep_smem_bytes(65536, 256)));
            if (pattr == cudaSuccess)
                pattr = cudaFuncSetAttribute(union_prep_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(prep_smem_bytes(65536, 256)));
            // the overlapped prep must use the gate GEMM's shared-memory carveout (the maximum), else an SM running a
            // gate GEMM CTA cannot also host a prep CTA
            if (pattr == cudaSuccess)
                pattr = cudaFuncSetAttribute(union_prep_kernel<true>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                             cudaSharedmemCarveoutMaxShared);
        });
        if (pattr != cudaSuccess) return SFFN_ERR_CUDA;
        const bool tma_dense = BR == 128 && N >= 256;
        // bits 16+: the work list orders each group's tiles by their fraction of the block's union (default; chunk-major
        // with SFFN_UP_ORDER=0) — ncu: 7B UP DRAM reads 2.0 -> 1.2 GB, 1.133 -> 1.105 ms; 70B 34 -> 21 GB, 9.54 -> 8.85 ms
        const int up_group = env_int("SFFN_UP_GROUP", union_group_up(NB, K)) |
                             (env_flag("SFFN_UP_ORDER", true) ? 1 << 16 : 0) | (env_flag("SFFN_UP_SNAKE", true) ? 2 << 16 : 0);
        const uint8_t* xin = gated ? static_cast<const uint8_t*>(X) : nullptr;
        uint8_t* xout = (gated && !env_flag("SFFN_PREP_NOCOPY", false)) ? static_cast<uint8_t*>(xp) : nullptr;
        int* pc = reinterpret_cast<int*>(base + L.pctr);
        const int dunits = union_dense_units(N, tma_dense);
        const int64_t dnnz = union_dense_nnz(N, tma_dense);
        unsigned long long* trace = prep_trace_buf(pctas);
        if (ovl) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(static_cast<unsigned>(pctas));
            cfg.blockDim = dim3(PREP_THREADS);
            cfg.dynamicSmemBytes = psmem;
            cfg.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = env_flag("SFFN_PREP_OV_NOPDL", false) ? 0 : 1;  // diagnostic: signals without the overlap
            if (cudaLaunchKernelEx(&cfg, union_prep_kernel<true>, tw, (int)M, (int)N, T, C, um, perm,
                                   static_cast<const int*>(rnnz), pc, up_group, split, boost, piece, ov, dunits, dnnz,
                                   xin, static_cast<int64_t>(K * 2), xout, gated ? 1 : 0, trace) != cudaSuccess)
                return SFFN_ERR_CUDA;
            note_launch();
        } else {
            union_prep_kernel<false><<<static_cast<unsigned>(pctas), PREP_THREADS, psmem, st>>>(
                tw, (int)M, (int)N, T, C, um, perm, rnnz, pc, up_group, split, boost, piece, ov, dunits, dnnz, xin,
                K * 2, xout, gated ? 1 : 0, trace);
            note_launch();
        }
        if (cudaGetLastError() != cudaSuccess) return SFFN_ERR_CUDA;
        if (!gated) {  // non-gated: H_c = the scattered TwELL values (no up GEMM)
            { union_gate_scatter_kernel<<<static_cast<unsigned>(NB * (BR / GS_ROWS)), 256, 0, st>>>(
                tw, (int)M, (int)N, T, C, um, static_cast<uint16_t*>(hc), perm); note_launch(); }
            if (cudaGetLastError() != cudaSuccess) return SFFN_ERR_CUDA;
        }
    }

    // operand maps: the single-CTA union GEMMs use k-blocks of UG_BK (SWIZZLE_64B K-major boxes at 32), the CTA-pair
    // kernels k-blocks of 64 (SWIZZLE_128B)
    const int kbk = BR == 256 ? GEMM_BK : UG_BK;
    const CUtensorMapSwizzle ksw = kbk == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
    CUtensorMap tx, twu, thc_st, thc_ld, twd, ty;
    if (!tmap_2d(&tx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, xp, K, M > 0 ? M : 1, kbk, GEMM_BM, ksw) ||
        !tmap_2d(&twu, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Wu, K, N, kbk, N >= 256 ? 256 : 64, ksw) ||
        !tmap_2d(&thc_st, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, hc, N, NB * BR, 64, 32, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !tmap_2d(&thc_ld, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, hc, N, NB * BR, kbk, GEMM_BM, ksw) ||
        !tmap_2d(&twd, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Wd, K, N, 64, kbk, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !tmap_2d(&ty, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Y, K, M, 128, 32, CU_TENSOR_MAP_SWIZZLE_NONE))
        return SFFN_ERR_CUDA;
    UnionArgs ua{};
    ua.M = (int)M;
    ua.K = (int)K;
    ua.N = (int)N;
    ua.T = T;
    ua.C = C;
    ua.NB = (int)NB;
    ua.NJ = (int)((K + 255) / 256);
    ua.group = env_int("SFFN_DOWN_GROUP", UNION_GROUP_DOWN);
    ua.tw = tw;
    ua.um = um;
    ua.perm = perm;
    ua.Y = static_cast<bf16_t*>(Y);
    ua.counter = um.counters;
    UnionArgs ud = ua;
    ud.counter = um.counters + 1;
    ua.wsrc = static_cast<const bf16_t*>(Wu);
    ud.wsrc = static_cast<const bf16_t*>(Wd);
    static std::once_flag once;
    static cudaError_t attr = cudaSuccess;
    std::call_once(once, [] {
        attr = cudaFuncSetAttribute(union_gemm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, UG_SMEM);
        if (attr == cudaSuccess)
            attr = cudaFuncSetAttribute(union_gemm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, UG_SMEM);
        if (attr == cudaSuccess)
            attr = cudaFuncSetAttribute(union_gemm_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        UG_SMEM);
        if (attr == cudaSuccess)
            attr = cudaFuncSetAttribute(union_gemm_pair_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        UGP_SMEM);
        if (attr == cudaSuccess)
            attr = cudaFuncSetAttribute(union_gemm_pair_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        UGP_SMEM);
    });
    if (attr != cudaSuccess) return SFFN_ERR_CUDA;
    const int sms = env_int("SFFN_UNION_GRID", dev_info().sms);  // tuning override (default: all SMs)
    const int64_t dtiles = NB * ua.NJ;
    if (BR == 256) {
        // CTA pairs: clusters of two, every role loop runs the same tile sequence in both CTAs
        auto launch_pair = [&](auto kern, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& o,
                               const UnionArgs& args, int64_t max_tiles) -> int {
            const int64_t pairs = std::min<int64_t>(max_tiles, sms / 2);
            if (pairs <= 0) return SFFN_OK;
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(static_cast<unsigned>(2 * pairs));
            cfg.blockDim = dim3(UG_THREADS);
            cfg.dynamicSmemBytes = UGP_SMEM;
            cfg.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 2;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            if (cudaLaunchKernelEx(&cfg, kern, a, b, o, args) != cudaSuccess) return SFFN_ERR_CUDA;
            note_launch();
            return SFFN_OK;
        };
        int r = SFFN_OK;
        if (gated && (r = launch_pair(union_gemm_pair_kernel<true>, tx, twu, thc_st, ua, sms)) != SFFN_OK) return r;
        if ((r = launch_pair(union_gemm_pair_kernel<false>, thc_ld, twd, ty, ud, dtiles)) != SFFN_OK) return r;
        return cudaGetLastError() == cudaSuccess ? SFFN_OK : SFFN_ERR_CUDA;
    }
    if (gated && phase != 2) {
        // UP: the number of (block, chunk) tiles is only known on the device; persistent grid.  For the
        // non-gated variant H_c already holds h = relu(x W_u) (the scattered TwELL values): no UP GEMM.
        { union_gemm_kernel<true><<<sms, UG_THREADS2, UG_SMEM, st>>>(tx, twu, thc_st, ua); note_launch(); }
        if (cudaGetLastError() != cudaSuccess) return SFFN_ERR_CUDA;
    }
    const int g2 = static_cast<int>(dtiles < sms ? dtiles : sms);
    if (phase == 1) return cudaGetLastError() == cudaSuccess ? SFFN_OK : SFFN_ERR_CUDA;
    if (fuse) {
        ud.ptrs = fuse->ptrs;
        ud.G = fuse->G;
        ud.rank = fuse->rank;
        { union_gemm_kernel<false, true><<<g2, UG_THREADS, UG_SMEM, st>>>(thc_ld, twd, ty, ud); note_launch(); }
    } else {
        { union_gemm_kernel<false><<<g2, UG_THREADS2, UG_SMEM, st>>>(thc_ld, twd, ty, ud); note_launch(); }
    }
    return cudaGetLastError() == cudaSuccess ? SFFN_OK : SFFN_ERR_CUDA;
}

int updown_dispatch(const void* X, const uint32_t* tw, const void* Wu, const void* Wd, int64_t M, int64_t K, int64_t N,
                    int T, int C, void* Y, void* ws, size_t ws_bytes, int algo, cudaStream_t st) {
    if (M == 0) return SFFN_OK;
    const int a = resolve_algo(algo, N);
    if (a == SFFN_ALGO_UNION) {
        if (!union_applicable(N)) return SFFN_ERR_SHAPE;
        if (!ws || ws_bytes < updown_ws_bytes(M, N, K, a, T, C)) return SFFN_ERR_SHAPE;
        return union_updown_impl(X, tw, Wu, Wd, M, K, N, T, C, Y, ws, st);
    }
    if (a != SFFN_ALGO_GATHER) return SFFN_ERR_INVALID_ARG;
    return updown_impl(X, tw, Wu, Wd, M, K, N, T, C, Y, st);
}

}  // namespace

extern "C" {

const char* sffn_status_string(int s) {
    switch (s) {
        case SFFN_OK: return "SFFN_OK";
        case SFFN_ERR_INVALID_ARG: return "SFFN_ERR_INVALID_ARG";
        case SFFN_ERR_SHAPE: return "SFFN_ERR_SHAPE";
        case SFFN_ERR_TILE_OVERFLOW: return "SFFN_ERR_TILE_OVERFLOW";
        case SFFN_ERR_CUDA: return "SFFN_ERR_CUDA";
        case SFFN_ERR_NCCL: return "SFFN_ERR_NCCL";
        case SFFN_ERR_UNSUPPORTED: return "SFFN_ERR_UNSUPPORTED";
    }
    return "SFFN_ERR_UNKNOWN";
}

int64_t sffn_launch_count(void) { return static_cast<int64_t>(g_launches.load()); }

const char* sffn_version(void) { return "sffn 0.1 (sm_100a tcgen05/TMEM/TMA)"; }

int64_t sffn_twell_words(int64_t M, int64_t N, int T, int C) {
    if (M < 0 || N < 0 || C <= 0 || T <= 0) return -1;
    (void)T;
    return M * (N / C);
}

size_t sffn_up_down_workspace_bytes(int64_t M, int64_t K, int64_t N, int T, int C, int algo) {
    if (M < 0 || N <= 0 || K <= 0 || !valid_TC(T, C)) return 0;
    return updown_ws_bytes(M, N, K, algo, T, C);
}

size_t sffn_forward_workspace_bytes(int64_t M, int64_t K, int64_t N, int T, int C, int algo) {
    int64_t w = sffn_twell_words(M, N, T, C);
    if (w < 0 || K <= 0) return 0;
    return static_cast<size_t>(align1k(w * 4)) + updown_ws_bytes(M, N, K, algo, T, C);
}

int sffn_pack(const void* X, const void* Wg, int64_t M, int64_t K, int64_t N, int T, int C, uint32_t* twell,
              uint32_t* d_overflow, void* stream) {
    int r = pack_checks(X, Wg, M, K, N, T, C, twell);
    if (r != SFFN_OK) return r;
    if ((r = check_device()) != SFFN_OK) return r;
    if (M == 0) return SFFN_OK;
    return pack_impl(X, Wg, M, K, N, T, C, twell, d_overflow, S(stream));
}

int sffn_unpack(const uint32_t* twell, int64_t M, int64_t N, int T, int C, int64_t col_offset, int64_t ld_dense,
                void* dense, void* stream) {
    if (!twell || !dense) return SFFN_ERR_INVALID_ARG;
    if (!valid_TC(T, C)) return SFFN_ERR_INVALID_ARG;
    if (M < 0 || N <= 0 || N % T != 0 || N > 65536 || col_offset < 0 || ld_dense < col_offset + N)
        return SFFN_ERR_SHAPE;
    int r = check_device();
    if (r != SFFN_OK) return r;
    const int64_t warps = M * (N / T);
    if (warps == 0) return SFFN_OK;
    const int64_t blocks = (warps * 32 + 255) / 256;
    if (blocks > 2147483647) return SFFN_ERR_SHAPE;
    { unpack_kernel<<<static_cast<unsigned>(blocks), 256, 0, S(stream)>>>(twell, (int)M, (int)N, T, C, col_offset,
                                                                         ld_dense, static_cast<__nv_bfloat16*>(dense)); note_launch(); }
    return cudaGetLastError() == cudaSuccess ? SFFN_OK : SFFN_ERR_CUDA;
}

int sffn_up_down(const void* X, const uint32_t* twell, const void* Wu, const void* Wd, int64_t M, int64_t K, int64_t N,
                 int T, int C, void* Y, void* workspace, size_t ws_bytes, int algo, void* stream) {
    if (algo < SFFN_ALGO_AUTO || algo > SFFN_ALGO_UNION) return SFFN_ERR_INVALID_ARG;
    int r = updown_checks(X, twell, Wu, Wd, M, K, N, T, C, Y, algo);
    if (r != SFFN_OK) return r;
    if (resolve_algo(algo, N) == SFFN_ALGO_UNION && M > 0) {
        if (!union_applicable(N)) return SFFN_ERR_SHAPE;
        if (!workspace || !aligned16(workspace) || ws_bytes < updown_ws_bytes(M, N, K, algo, T, C)) return SFFN_ERR_SHAPE;
    }
    if ((r = check_device()) != SFFN_OK) return r;
    return updown_dispatch(X, twell, Wu, Wd, M, K, N, T, C, Y, workspace, ws_bytes, algo, S(stream));
}

int sffn_forward(const void* X, const void* Wg, const void* Wu, const void* Wd, int64_t M, int64_t K, int64_t N, int T,
                 int C, void* Y, void* workspace, size_t ws_bytes, uint32_t* d_overflow, int algo, void* stream) {
    int r = pack_checks(X, Wg, M, K, N, T, C, workspace);
    if (r != SFFN_OK) return r;
    if (algo < SFFN_ALGO_AUTO || algo > SFFN_ALGO_UNION) return SFFN_ERR_INVALID_ARG;
    if ((r = updown_checks(X, workspace, Wu, Wd, M, K, N, T, C, Y, algo)) != SFFN_OK) return r;
    if (resolve_algo(algo, N) == SFFN_ALGO_UNION && !union_applicable(N)) return SFFN_ERR_SHAPE;
    if (ws_bytes < sffn_forward_workspace_bytes(M, K, N, T, C, algo)) return SFFN_ERR_SHAPE;
    if ((r = check_device()) != SFFN_OK) return r;
    if (M == 0) return SFFN_OK;
    uint32_t* tw = static_cast<uint32_t*>(workspace);
    const int64_t tw_bytes = align1k(sffn_twell_words(M, N, T, C) * 4);
    uint8_t* udws = static_cast<uint8_t*>(workspace) + tw_bytes;
    if (resolve_algo(algo, N) == SFFN_ALGO_UNION) {
        // the gate GEMM epilogue also counts each row's stored entries (the union path's row order pi)
        int* nnz = union_nnz_ptr(udws, M, N, K, T, C);
        if (cudaMemsetAsync(nnz, 0, union_zero_bytes(M, N, K, T, C), S(stream)) != cudaSuccess) return SFFN_ERR_CUDA;
        // overlapped prep: CTA-pair gate GEMM, 128-row union blocks, and room for a prep CTA beside a gate GEMM CTA
        static const bool gate_pair = env_flag("SFFN_GATE_PAIR", true);
        const UnionWs L = union_ws_layout(M, N, K, T, C);
        const int ov_piece = (union_prep_overlap_enabled() && gate_pair && union_brows() == 128)
                                 ? prep_overlap_piece(N, L.nchunk, C) : 0;
        int* win_done = ov_piece > 0 ? reinterpret_cast<int*>(udws + L.pctr) + 2 + 2 * ((M + 127) / 128) : nullptr;
        if ((r = pack_impl(X, Wg, M, K, N, T, C, tw, d_overflow, S(stream), nnz, nnz + M, win_done)) != SFFN_OK) return r;
        return union_updown_impl(X, tw, Wu, Wd, M, K, N, T, C, Y, udws, S(stream), true, true, nullptr, ov_piece);
    }
    if ((r = pack_impl(X, Wg, M, K, N, T, C, tw, d_overflow, S(stream))) != SFFN_OK) return r;
    return updown_dispatch(X, tw, Wu, Wd, M, K, N, T, C, Y, udws, ws_bytes - static_cast<size_t>(tw_bytes), algo,
                           S(stream));
}

// Internal (not in include/sffn.h): sffn_forward (UNION) whose DOWN GEMM writes the partial Y into this rank's
// symmetric window (Y) and reduces 2048-row windows across the ranks as they complete (sffn_comm.cu).
// Internal (tools): the prep kernel's per-CTA phase timestamps of the last traced call (SFFN_PREP_TRACE=1).
#ifdef SFFN_GEMM_EPI_TRACE
// Internal (probe builds): the gate GEMM role cycle sums (g_gemm_trace), copied out and reset
int sffn__gemm_trace(unsigned long long* host) {
    if (cudaMemcpyFromSymbol(host, g_gemm_trace, sizeof(unsigned long long) * 8) != cudaSuccess) return -1;
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    return cudaMemcpyToSymbol(g_gemm_trace, z, sizeof(z)) == cudaSuccess ? 0 : -1;
}
#endif
int64_t sffn__prep_trace(unsigned long long* host, int64_t cap) {
    if (!g_prep_trace) return 0;
    const int64_t n = cap < g_prep_trace_n ? cap : g_prep_trace_n;
    if (cudaMemcpy(host, g_prep_trace, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    return n;
}

int sffn__forward_fused(const void* X, const void* Wg, const void* Wu, const void* Wd, int64_t M, int64_t K, int64_t N,
                        int T, int C, void* Y, void* workspace, size_t ws_bytes, uint32_t* d_overflow,
                        const uint64_t* ptrs, int G, int rank, int phase, void* stream) {
    int r = pack_checks(X, Wg, M, K, N, T, C, workspace);
    if (r != SFFN_OK) return r;
    if ((r = updown_checks(X, workspace, Wu, Wd, M, K, N, T, C, Y, SFFN_ALGO_UNION)) != SFFN_OK) return r;
    if (!union_applicable(N) || union_brows() != 128) return SFFN_ERR_UNSUPPORTED;
    if (ws_bytes < sffn_forward_workspace_bytes(M, K, N, T, C, SFFN_ALGO_UNION)) return SFFN_ERR_SHAPE;
    if ((r = check_device()) != SFFN_OK) return r;
    if (M == 0) return SFFN_OK;
    if (phase < 0 || phase > 2) return SFFN_ERR_INVALID_ARG;
    uint32_t* tw = static_cast<uint32_t*>(workspace);
    const int64_t tw_bytes = align1k(sffn_twell_words(M, N, T, C) * 4);
    uint8_t* udws = static_cast<uint8_t*>(workspace) + tw_bytes;
    int* nnz = union_nnz_ptr(udws, M, N, K, T, C);
    FuseParams fp{ptrs, G, rank, phase};
    if (phase == 2) return union_updown_impl(X, tw, Wu, Wd, M, K, N, T, C, Y, udws, S(stream), true, true, &fp);
    if (cudaMemsetAsync(nnz, 0, union_zero_bytes(M, N, K, T, C), S(stream)) != cudaSuccess) return SFFN_ERR_CUDA;
    if ((r = pack_impl(X, Wg, M, K, N, T, C, tw, d_overflow, S(stream), nnz, nnz + M)) != SFFN_OK) return r;
    return union_updown_impl(X, tw, Wu, Wd, M, K, N, T, C, Y, udws, S(stream), true, true, &fp);
}

int sffn_down(const uint32_t* twell, const void* Wd, int64_t M, int64_t K, int64_t N, int T, int C, void* Y,
              void* workspace, size_t ws_bytes, int algo, void* stream) {
    if (algo < SFFN_ALGO_AUTO || algo > SFFN_ALGO_UNION) return SFFN_ERR_INVALID_ARG;
    int r = updown_checks(Wd, twell, Wd, Wd, M, K, N, T, C, Y, algo);
    if (r != SFFN_OK) return r;
    const int a = resolve_algo(algo, N);
    if (a == SFFN_ALGO_UNION && M > 0) {
        if (!union_applicable(N)) return SFFN_ERR_SHAPE;
        if (!workspace || !aligned16(workspace) || ws_bytes < updown_ws_bytes(M, N, K, a, T, C)) return SFFN_ERR_SHAPE;
    }
    if ((r = check_device()) != SFFN_OK) return r;
    if (M == 0) return SFFN_OK;
    cudaStream_t st = S(stream);
    if (a == SFFN_ALGO_UNION) return union_updown_impl(Wd, twell, Wd, Wd, M, K, N, T, C, Y, workspace, st, false);
    const int64_t per_warp = (K / 8 + UD_WARPS - 1) / UD_WARPS;
    const int nch = static_cast<int>((per_warp + 31) / 32);
    const uint4* wd = static_cast<const uint4*>(Wd);
    uint4* y = static_cast<uint4*>(Y);
    dim3 g(static_cast<unsigned>(M)), blk(UD_WARPS * 32);
    if (nch <= 1) { down_kernel<1><<<g, blk, 0, st>>>(twell, wd, y, (int)M, (int)K, (int)N, T, C); note_launch(); }
    else if (nch <= 2) { down_kernel<2><<<g, blk, 0, st>>>(twell, wd, y, (int)M, (int)K, (int)N, T, C); note_launch(); }
    else if (nch <= 4) { down_kernel<4><<<g, blk, 0, st>>>(twell, wd, y, (int)M, (int)K, (int)N, T, C); note_launch(); }
    else if (nch <= 8) { down_kernel<8><<<g, blk, 0, st>>>(twell, wd, y, (int)M, (int)K, (int)N, T, C); note_launch(); }
    else return SFFN_ERR_SHAPE;
    return cudaGetLastError() == cudaSuccess ? SFFN_OK : SFFN_ERR_CUDA;
}

int sffn_forward_nongated(const void* X, const void* Wu, const void* Wd, int64_t M, int64_t K, int64_t N, int T, int C,
                          void* Y, void* workspace, size_t ws_bytes, uint32_t* d_overflow, int algo, void* stream) {
    int r = pack_checks(X, Wu, M, K, N, T, C, workspace);
    if (r != SFFN_OK) return r;
    if (ws_bytes < sffn_forward_workspace_bytes(M, K, N, T, C, algo)) return SFFN_ERR_SHAPE;
    if ((r = check_device()) != SFFN_OK) return r;
    if (M == 0) return SFFN_OK;
    uint32_t* tw = static_cast<uint32_t*>(workspace);
    const int64_t tw_bytes = align1k(sffn_twell_words(M, N, T, C) * 4);
    if ((r = pack_impl(X, Wu, M, K, N, T, C, tw, d_overflow, S(stream))) != SFFN_OK) return r;
    return sffn_down(tw, Wd, M, K, N, T, C, Y, static_cast<uint8_t*>(workspace) + tw_bytes,
                     ws_bytes - static_cast<size_t>(tw_bytes), algo, stream);
}

int sffn_dense_forward(const void* X, const void* Wg, const void* Wu, const void* WdT, int64_t M, int64_t K, int64_t N,
                       void* H, void* Y, void* stream) {
    if (!X || !Wg || !Wu || !WdT || !H || !Y) return SFFN_ERR_INVALID_ARG;
    if (!aligned16(X) || !aligned16(Wg) || !aligned16(Wu) || !aligned16(WdT) || !aligned16(H) || !aligned16(Y))
        return SFFN_ERR_INVALID_ARG;
    if (M < 0 || K < 64 || K % 64 != 0 || N < 128 || N % 128 != 0) return SFFN_ERR_SHAPE;
    if (M > (int64_t(1) << 31) - GEMM_BM || K > (int64_t(1) << 30) || N > (int64_t(1) << 30)) return SFFN_ERR_SHAPE;
    int r = check_device();
    if (r != SFFN_OK) return r;
    if (M == 0) return SFFN_OK;
    static const bool pair = env_flag("SFFN_GATE_PAIR", true);
    CUtensorMap tx, tg, tu, th_out, th_in, twd, ty;
    if (!tmap_2d(&tx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, X, K, M, GEMM_BK, GEMM_BM, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !tmap_2d(&tg, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Wg, K, N, GEMM_BK, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !tmap_2d(&tu, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Wu, K, N, GEMM_BK, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !tmap_2d(&th_out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, H, N, M, 128, 32, CU_TENSOR_MAP_SWIZZLE_NONE) ||
        !tmap_2d(&th_in, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, H, N, M, GEMM_BK, GEMM_BM, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !tmap_2d(&twd, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, WdT, N, K, GEMM_BK, pair ? GEMM_BN / 2 : GEMM_BN,
                 CU_TENSOR_MAP_SWIZZLE_128B) ||
        !tmap_2d(&ty, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Y, K, M, 128, 32, CU_TENSOR_MAP_SWIZZLE_NONE))
        return SFFN_ERR_CUDA;
    GemmArgs a1{};
    a1.M = (int)M;
    a1.N = (int)N;
    a1.K = (int)K;
    GemmArgs a2{};
    a2.M = (int)M;
    a2.N = (int)K;
    a2.K = (int)N;
    // CTA pairs like the gate GEMM (the GLU tile's W_g half on one CTA, its W_u half on the other): the
    // speedup denominator uses the same tcgen05 machinery as the sparse path
    if (pair) {
        if ((r = launch_gemm<EPI_GLU, 1, 2>(tx, tg, tu, th_out, a1, 128, S(stream))) != SFFN_OK) return r;
        return launch_gemm<EPI_BF16, 1, 2>(th_in, twd, twd, ty, a2, GEMM_BN, S(stream));
    }
    if ((r = launch_gemm<EPI_GLU, 1>(tx, tg, tu, th_out, a1, 128, S(stream))) != SFFN_OK) return r;
    return launch_gemm<EPI_BF16, 1>(th_in, twd, twd, ty, a2, GEMM_BN, S(stream));
}

int sffn_transpose_bf16(const void* in, int64_t rows, int64_t cols, void* out, void* stream) {
    if (!in || !out) return SFFN_ERR_INVALID_ARG;
    if (rows < 0 || cols < 0 || (rows + 31) / 32 > 65535) return SFFN_ERR_SHAPE;
    int r = check_device();
    if (r != SFFN_OK) return r;
    if (rows == 0 || cols == 0) return SFFN_OK;
    dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((rows + 31) / 32)), block(32, 8);
    { transpose_bf16_kernel<<<grid, block, 0, S(stream)>>>(static_cast<const __nv_bfloat16*>(in), rows, cols,
                                                         static_cast<__nv_bfloat16*>(out)); note_launch(); }
    return cudaGetLastError() == cudaSuccess ? SFFN_OK : SFFN_ERR_CUDA;
}

int sffn_gate_gemm_f32(const void* X, const void* Wg, int64_t M, int64_t K, int64_t N, float* Sout, void* stream) {
    if (!X || !Wg || !Sout) return SFFN_ERR_INVALID_ARG;
    if (!aligned16(X) || !aligned16(Wg) || !aligned16(Sout)) return SFFN_ERR_INVALID_ARG;
    if (M < 0 || K < 64 || K % 64 != 0 || N <= 0 || N % 16 != 0) return SFFN_ERR_SHAPE;
    if (M > (int64_t(1) << 31) - GEMM_BM || N > (int64_t(1) << 30)) return SFFN_ERR_SHAPE;
    int r = check_device();
    if (r != SFFN_OK) return r;
    if (M == 0) return SFFN_OK;
    // the same mainloop as the pack (CTA pairs unless SFFN_GATE_PAIR=0): verifies the production accumulators
    static const bool pair = env_flag("SFFN_GATE_PAIR", true);
    CUtensorMap ta, tb;
    if (!tmap_2d(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, X, K, M, GEMM_BK, GEMM_BM, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !tmap_2d(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Wg, K, N, GEMM_BK, pair ? GEMM_BN / 2 : GEMM_BN,
                 CU_TENSOR_MAP_SWIZZLE_128B))
        return SFFN_ERR_CUDA;
    GemmArgs args{};
    args.M = (int)M;
    args.N = (int)N;
    args.K = (int)K;
    args.out_f32 = Sout;
    args.ld_out = N;
    return pair ? launch_gemm<EPI_F32, 1, 2>(ta, tb, tb, tb, args, GEMM_BN, S(stream))
                : launch_gemm<EPI_F32, 1>(ta, tb, tb, tb, args, GEMM_BN, S(stream));
}

// ---------------------------------------------------------------- fp32 mode (R19)
struct F32Ws {
    int64_t hv, hi, hnz, total;
};
static F32Ws f32_layout(int64_t M, int64_t N, int T, int C) {
    F32Ws w{};
    w.hv = 0;
    w.hi = align1k(M * (N / C) * 4);
    w.hnz = w.hi + align1k(M * (N / C) * 2);
    w.total = w.hnz + align1k(M * (N / T) * 4);
    return w;
}

size_t sffn_f32_twell_bytes(int64_t M, int64_t N, int T, int C) {
    if (M < 0 || N <= 0 || !valid_TC(T, C)) return 0;
    return static_cast<size_t>(f32_layout(M, N, T, C).total);
}

int sffn_pack_f32(const float* X, const float* Wg, int64_t M, int64_t K, int64_t N, int T, int C, float* hv,
                  uint16_t* hi, uint32_t* hnz, uint32_t* d_overflow, void* stream) {
    if (M == 0 && valid_TC(T, C)) return SFFN_OK;
    if (!X || !Wg || !hv || !hi || !hnz) return SFFN_ERR_INVALID_ARG;
    if (!valid_TC(T, C)) return SFFN_ERR_INVALID_ARG;
    if (M < 0 || K < 4 || K % 4 != 0 || N <= 0 || N % T != 0 || N > 65536 || M > 2147483647) return SFFN_ERR_SHAPE;
    int r = check_device();
    if (r != SFFN_OK) return r;
    const int smem = F32_BM * (F32_BN + 1) * 4;
    static std::once_flag once;
    static cudaError_t attr = cudaSuccess;
    std::call_once(once, [&] { attr = cudaFuncSetAttribute(pack_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); });
    if (attr != cudaSuccess) return SFFN_ERR_CUDA;
    dim3 grid(static_cast<unsigned>((N + F32_BN - 1) / F32_BN), static_cast<unsigned>((M + F32_BM - 1) / F32_BM));
    if (grid.y > 65535) return SFFN_ERR_SHAPE;
    { pack_f32_kernel<<<grid, 256, smem, S(stream)>>>(X, Wg, (int)M, (int)K, (int)N, T, C, hv, hi, hnz, d_overflow); note_launch(); }
    return cudaGetLastError() == cudaSuccess ? SFFN_OK : SFFN_ERR_CUDA;
}

int sffn_up_down_f32(const float* X, const float* hv, const uint16_t* hi, const uint32_t* hnz, const float* Wu,
                     const float* Wd, int64_t M, int64_t K, int64_t N, int T, int C, float* Y, void* stream) {
    if (M == 0 && valid_TC(T, C)) return SFFN_OK;
    if (!X || !hv || !hi || !hnz || !Wu || !Wd || !Y) return SFFN_ERR_INVALID_ARG;
    if (!aligned16(X) || !aligned16(Wu) || !aligned16(Wd) || !aligned16(Y)) return SFFN_ERR_INVALID_ARG;
    if (!valid_TC(T, C)) return SFFN_ERR_INVALID_ARG;
    if (M < 0 || K < 4 || K % 4 != 0 || K > 8192 || N <= 0 || N % T != 0 || N > 65536 || M > 2147483647)
        return SFFN_ERR_SHAPE;
    int r = check_device();
    if (r != SFFN_OK) return r;
    const int64_t per_warp = (K / 4 + 3) / 4;
    const int nch = static_cast<int>((per_warp + 31) / 32);
    const float4* x = reinterpret_cast<const float4*>(X);
    const float4* wu = reinterpret_cast<const float4*>(Wu);
    const float4* wd = reinterpret_cast<const float4*>(Wd);
    float4* y = reinterpret_cast<float4*>(Y);
    dim3 g(static_cast<unsigned>(M));
    cudaStream_t st = S(stream);
    if (nch <= 1) { updown_f32_kernel<1><<<g, 128, 0, st>>>(x, hv, hi, hnz, wu, wd, y, (int)M, (int)K, (int)N, T, C); note_launch(); }
    else if (nch <= 2) { updown_f32_kernel<2><<<g, 128, 0, st>>>(x, hv, hi, hnz, wu, wd, y, (int)M, (int)K, (int)N, T, C); note_launch(); }
    else if (nch <= 4) { updown_f32_kernel<4><<<g, 128, 0, st>>>(x, hv, hi, hnz, wu, wd, y, (int)M, (int)K, (int)N, T, C); note_launch(); }
    else if (nch <= 8) { updown_f32_kernel<8><<<g, 128, 0, st>>>(x, hv, hi, hnz, wu, wd, y, (int)M, (int)K, (int)N, T, C); note_launch(); }
    else { updown_f32_kernel<16><<<g, 128, 0, st>>>(x, hv, hi, hnz, wu, wd, y, (int)M, (int)K, (int)N, T, C); note_launch(); }
    return cudaGetLastError() == cudaSuccess ? SFFN_OK : SFFN_ERR_CUDA;
}

int sffn_forward_f32(const float* X, const float* Wg, const float* Wu, const float* Wd, int64_t M, int64_t K, int64_t N,
                     int T, int C, float* Y, void* workspace, size_t ws_bytes, uint32_t* d_overflow, void* stream) {
    if (!valid_TC(T, C)) return SFFN_ERR_INVALID_ARG;
    if (M < 0 || N <= 0) return SFFN_ERR_SHAPE;
    if (M == 0) return SFFN_OK;
    if (!workspace || !aligned16(workspace)) return SFFN_ERR_INVALID_ARG;
    if (ws_bytes < sffn_f32_twell_bytes(M, N, T, C)) return SFFN_ERR_SHAPE;
    F32Ws L = f32_layout(M, N, T, C);
    uint8_t* b = static_cast<uint8_t*>(workspace);
    float* hv = reinterpret_cast<float*>(b + L.hv);
    uint16_t* hi = reinterpret_cast<uint16_t*>(b + L.hi);
    uint32_t* hnz = reinterpret_cast<uint32_t*>(b + L.hnz);
    int r = sffn_pack_f32(X, Wg, M, K, N, T, C, hv, hi, hnz, d_overflow, stream);
    if (r != SFFN_OK) return r;
    return sffn_up_down_f32(X, hv, hi, hnz, Wu, Wd, M, K, N, T, C, Y, stream);
}

// ---------------------------------------------------------------- host-buffer forward (copy/compute overlap)
namespace {
struct CopyStreams {
    cudaStream_t h2d = nullptr, d2h = nullptr, comp = nullptr;  // comp: second compute stream of forward_host
};
std::mutex g_cs_mu;
CopyStreams g_cs[64];
int copy_streams(int dev, CopyStreams* out) {
    if (dev < 0 || dev >= 64) return SFFN_ERR_UNSUPPORTED;
    std::lock_guard<std::mutex> lk(g_cs_mu);
    CopyStreams& c = g_cs[dev];
    if (!c.h2d) {
        if (cudaStreamCreateWithFlags(&c.h2d, cudaStreamNonBlocking) != cudaSuccess) return SFFN_ERR_CUDA;
        if (cudaStreamCreateWithFlags(&c.d2h, cudaStreamNonBlocking) != cudaSuccess) return SFFN_ERR_CUDA;
        if (cudaStreamCreateWithFlags(&c.comp, cudaStreamNonBlocking) != cudaSuccess) return SFFN_ERR_CUDA;
    }
    *out = c;
    return SFFN_OK;
}
}  // namespace

// Row chunks of sffn_forward_host: sizes ramp geometrically (R/4, R/2, ...) up to R = chunk_rows at the start and
// back down at the end, so the first host->device copy and the last device->host copy (pipeline fill and drain,
// not overlapped with compute) are short, while the middle chunks are large (the per-call fixed cost of the
// forward is amortised).  Chunk starts stay multiples of the unit u (2048 when R is, so the UNION permutation
// windows are those of one sffn_forward call); a ragged remainder goes to the last chunk.  Every size <= R.
// (A finer ramp — 512, 1024, 2048 at both ends, SFFN_HOST_RAMP_MIN=512 — measured 7.31 vs 6.75 ms at 7B: the
// extra chunks' fixed costs outweigh the shorter fill.)
static std::vector<int64_t> host_chunk_plan(int64_t M, int64_t R) {
    std::vector<int64_t> out;
    static const int64_t rmin = std::max<int64_t>(128, env_int("SFFN_HOST_RAMP_MIN", 2048) / 128 * 128);
    const int64_t u = R % rmin == 0 ? rmin : 128;
    std::vector<int64_t> ramp;
    for (int64_t s = std::max(u, (R / (rmin < 2048 ? 8 : 4)) / u * u); s < R; s *= 2) ramp.push_back(s);
    int64_t rsum = 0;
    for (int64_t s : ramp) rsum += s;
    const int64_t Mu = M / u * u;
    if (ramp.empty() || 2 * rsum >= Mu || M - Mu + ramp.front() > R) {
        for (int64_t r0 = 0; r0 < M; r0 += R) out.push_back(std::min(R, M - r0));
        return out;
    }
    const int64_t mid = Mu - 2 * rsum;
    const int64_t n = (mid + R - 1) / R;
    const int64_t each = ((mid / n) + u - 1) / u * u;
    out = ramp;
    int64_t left = mid;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t s = i + 1 < n ? std::min(each, left) : left;
        out.push_back(s);
        left -= s;
    }
    for (auto it = ramp.rbegin(); it != ramp.rend(); ++it) out.push_back(*it);
    out.back() += M - Mu;
    return out;
}

int64_t sffn_forward_host_chunks(int64_t M, int64_t chunk_rows, int64_t* sizes, int64_t cap) {
    if (M <= 0 || chunk_rows <= 0 || chunk_rows % 128 != 0) return 0;
    const int64_t rows = chunk_rows < M ? chunk_rows : ((M + 127) / 128) * 128;
    std::vector<int64_t> v = host_chunk_plan(M, rows);
    for (int64_t i = 0; sizes && i < cap && i < static_cast<int64_t>(v.size()); ++i) sizes[i] = v[static_cast<size_t>(i)];
    return static_cast<int64_t>(v.size());
}

// X / Y staging slots of sffn_forward_host (double buffering; 3 slots measured 1% slower at 4096-row chunks)
constexpr int HOST_SLOTS = 2;

size_t sffn_forward_host_stage_bytes(int64_t K, int64_t chunk_rows) {
    if (K <= 0 || chunk_rows <= 0) return 0;
    return static_cast<size_t>(2 * HOST_SLOTS * align1k(chunk_rows * K * 2));  // HOST_SLOTS X slots + HOST_SLOTS Y
}

int sffn_forward_host(const void* X_host, const void* Wg, const void* Wu, const void* Wd, int64_t M, int64_t K,
                      int64_t N, int T, int C, void* Y_host, void* workspace, size_t ws_bytes, void* stage,
                      size_t stage_bytes, uint32_t* d_overflow, int algo, int64_t chunk_rows, void* stream) {
    if (!X_host || !Y_host || !stage) return M == 0 ? SFFN_OK : SFFN_ERR_INVALID_ARG;
    if (chunk_rows <= 0 || chunk_rows % 128 != 0) return SFFN_ERR_SHAPE;
    if (M < 0 || K <= 0) return SFFN_ERR_SHAPE;
    if (M == 0) return SFFN_OK;
    const int64_t rows = chunk_rows < M ? chunk_rows : ((M + 127) / 128) * 128;
    if (stage_bytes < sffn_forward_host_stage_bytes(K, rows)) return SFFN_ERR_SHAPE;
    const size_t wsz = sffn_forward_workspace_bytes(rows < M ? rows : M, K, N, T, C, algo);
    if (ws_bytes < wsz) return SFFN_ERR_SHAPE;
    int r = check_device();
    if (r != SFFN_OK) return r;
    int dev = 0;
    cudaGetDevice(&dev);
    CopyStreams cs;
    if ((r = copy_streams(dev, &cs)) != SFFN_OK) return r;
    cudaStream_t st = S(stream);
    // two workspaces -> consecutive chunks compute on two streams (`stream` and an internal one), so the kernels of
    // chunk i+1 start on the SMs that chunk i's persistent kernels release in their tails
    const size_t wsz1k = static_cast<size_t>(align1k(static_cast<int64_t>(wsz)));
    const bool dual = ws_bytes >= wsz1k + wsz;
    cudaStream_t cst[2] = {st, dual ? cs.comp : st};
    uint8_t* wss[2] = {static_cast<uint8_t*>(workspace), static_cast<uint8_t*>(workspace) + (dual ? wsz1k : 0)};
    // chunk schedule: ramp up / down in size at the ends (short pipeline fill and drain), full chunks between
    std::vector<int64_t> sizes = host_chunk_plan(M, rows);
    const int64_t nchunks = static_cast<int64_t>(sizes.size());
    const int64_t slot = align1k(rows * K * 2);
    // staging slots: HOST_SLOTS by default; a larger stage buffer buys more (up to one per chunk), so a copy never
    // waits for a slot still in use by a chunk two places back
    const int64_t nslots = std::max<int64_t>(HOST_SLOTS, std::min<int64_t>(nchunks, static_cast<int64_t>(stage_bytes) / (2 * slot)));
    std::vector<uint8_t*> xs(static_cast<size_t>(nslots)), ys(static_cast<size_t>(nslots));
    for (int64_t q = 0; q < nslots; ++q) {
        xs[static_cast<size_t>(q)] = static_cast<uint8_t*>(stage) + q * slot;
        ys[static_cast<size_t>(q)] = static_cast<uint8_t*>(stage) + (nslots + q) * slot;
    }
    // events: per chunk h2d done, compute done, d2h done
    std::vector<cudaEvent_t> ev(static_cast<size_t>(3 * nchunks + 1));
    for (auto& e : ev)
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return SFFN_ERR_CUDA;
    auto E = [&](int kind, int64_t i) { return ev[static_cast<size_t>(3 * i + kind)]; };
    // the copies must not start before earlier work on `stream`
    cudaEventRecord(ev.back(), st);
    cudaStreamWaitEvent(cs.h2d, ev.back(), 0);
    cudaStreamWaitEvent(cs.d2h, ev.back(), 0);
    if (dual) cudaStreamWaitEvent(cs.comp, ev.back(), 0);
    int64_t r0 = 0;
    for (int64_t i = 0; i < nchunks && r == SFFN_OK; r0 += sizes[static_cast<size_t>(i)], ++i) {
        const int64_t mr = sizes[static_cast<size_t>(i)];
        const size_t bytes = static_cast<size_t>(mr * K * 2);
        const size_t sl = static_cast<size_t>(i % nslots);
        if (i >= nslots) cudaStreamWaitEvent(cs.h2d, E(1, i - nslots), 0);  // X slot free: chunk computed
        if (cudaMemcpyAsync(xs[sl], static_cast<const uint8_t*>(X_host) + r0 * K * 2, bytes, cudaMemcpyHostToDevice,
                            cs.h2d) != cudaSuccess) { r = SFFN_ERR_CUDA; break; }
        cudaEventRecord(E(0, i), cs.h2d);
        const int cw = static_cast<int>(i & 1);  // compute stream / workspace half: chunk i-2 used it, ordered
        cudaStream_t cs_i = cst[cw];
        cudaStreamWaitEvent(cs_i, E(0, i), 0);
        if (i >= nslots) cudaStreamWaitEvent(cs_i, E(2, i - nslots), 0);  // Y slot free: chunk copied out
        r = sffn_forward(xs[sl], Wg, Wu, Wd, mr, K, N, T, C, ys[sl], wss[cw], wsz, d_overflow, algo, cs_i);
        if (r != SFFN_OK) break;
        cudaEventRecord(E(1, i), cs_i);
        cudaStreamWaitEvent(cs.d2h, E(1, i), 0);
        if (cudaMemcpyAsync(static_cast<uint8_t*>(Y_host) + r0 * K * 2, ys[sl], bytes, cudaMemcpyDeviceToHost,
                            cs.d2h) != cudaSuccess) { r = SFFN_ERR_CUDA; break; }
        cudaEventRecord(E(2, i), cs.d2h);
    }
    if (r == SFFN_OK) {
        cudaEventRecord(ev.back(), cs.d2h);
        cudaStreamWaitEvent(st, ev.back(), 0);  // the call completes on `stream`
    }
    for (auto& e : ev) cudaEventDestroy(e);  // destruction is deferred until the events complete
    return r;
}

// ---------------------------------------------------------------- overflow-exact (hybrid) forward
namespace {
struct HybWs {
    int64_t fwd, cnt, list, xo, ho, yo, total;
};
HybWs hyb_layout(int64_t M, int64_t K, int64_t N, int T, int C, int algo, int64_t R) {
    HybWs w{};
    w.fwd = 0;
    int64_t o = align1k(static_cast<int64_t>(sffn_forward_workspace_bytes(M, K, N, T, C, algo)));
    w.cnt = o;  o = align1k(o + 16);
    w.list = o; o = align1k(o + R * 4);
    w.xo = o;   o = align1k(o + R * K * 2);
    w.ho = o;   o = align1k(o + R * N * 2);
    w.yo = o;   o = align1k(o + R * K * 2);
    w.total = o;
    return w;
}
}  // namespace

size_t sffn_hybrid_workspace_bytes(int64_t M, int64_t K, int64_t N, int T, int C, int algo, int64_t backup_rows) {
    if (M < 0 || K <= 0 || N <= 0 || backup_rows < 0) return 0;
    const int64_t R = ((backup_rows + 127) / 128) * 128;
    return static_cast<size_t>(hyb_layout(M, K, N, T, C, algo, R).total);
}

int sffn_forward_hybrid(const void* X, const void* Wg, const void* Wu, const void* Wd, int64_t M, int64_t K, int64_t N,
                        int T, int C, void* Y, void* workspace, size_t ws_bytes, int64_t backup_rows,
                        int* d_backup_count, uint32_t* d_overflow, int algo, void* stream) {
    if (backup_rows < 0) return SFFN_ERR_INVALID_ARG;
    if (N % 128 != 0) return SFFN_ERR_SHAPE;  // dense backup GEMM tiles
    const int64_t R = ((backup_rows + 127) / 128) * 128;
    if (ws_bytes < sffn_hybrid_workspace_bytes(M, K, N, T, C, algo, backup_rows)) return SFFN_ERR_SHAPE;
    HybWs L = hyb_layout(M, K, N, T, C, algo, R);
    uint8_t* b = static_cast<uint8_t*>(workspace);
    int r = sffn_forward(X, Wg, Wu, Wd, M, K, N, T, C, Y, b, static_cast<size_t>(L.cnt), d_overflow, algo, stream);
    if (r != SFFN_OK || M == 0) return r;
    cudaStream_t st = S(stream);
    int* cnt = reinterpret_cast<int*>(b + L.cnt);
    int32_t* list = reinterpret_cast<int32_t*>(b + L.list);
    if (cudaMemsetAsync(cnt, 0, 4, st) != cudaSuccess) return SFFN_ERR_CUDA;
    { ov_rows_kernel<<<static_cast<unsigned>((M * 32 + 255) / 256), 256, 0, st>>>(
        static_cast<const uint32_t*>(workspace), (int)M, (int)N, T, C, cnt, list, (int)R); note_launch(); }
    if (cudaGetLastError() != cudaSuccess) return SFFN_ERR_CUDA;
    if (d_backup_count && cudaMemcpyAsync(d_backup_count, cnt, 4, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return SFFN_ERR_CUDA;
    if (R == 0) return SFFN_OK;
    void* xo = b + L.xo;
    void* ho = b + L.ho;
    void* yo = b + L.yo;
    const unsigned g = static_cast<unsigned>((R * 32 + 255) / 256);
    { move_rows_kernel<true><<<g, 256, 0, st>>>(static_cast<const uint4*>(X), static_cast<uint4*>(xo), list, cnt, (int)R,
                                              (int)(K / 8)); note_launch(); }
    if (cudaGetLastError() != cudaSuccess) return SFFN_ERR_CUDA;
    CUtensorMap tx, tg, tu, th_out, th_in, twd, ty;
    if (!tmap_2d(&tx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, xo, K, R, GEMM_BK, GEMM_BM, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !tmap_2d(&tg, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Wg, K, N, GEMM_BK, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !tmap_2d(&tu, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Wu, K, N, GEMM_BK, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !tmap_2d(&th_out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ho, N, R, 128, 32, CU_TENSOR_MAP_SWIZZLE_NONE) ||
        !tmap_2d(&th_in, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ho, N, R, GEMM_BK, GEMM_BM, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !tmap_2d(&twd, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Wd, K, N, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !tmap_2d(&ty, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, yo, K, R, 128, 32, CU_TENSOR_MAP_SWIZZLE_NONE))
        return SFFN_ERR_CUDA;
    GemmArgs a1{};
    a1.M = (int)R;
    a1.N = (int)N;
    a1.K = (int)K;
    a1.m_dev = cnt;
    if ((r = launch_gemm<EPI_GLU, 1>(tx, tg, tu, th_out, a1, 128, st)) != SFFN_OK) return r;
    GemmArgs a2{};
    a2.M = (int)R;
    a2.N = (int)K;
    a2.K = (int)N;
    a2.m_dev = cnt;
    if ((r = launch_gemm<EPI_BF16_MN, 1>(th_in, twd, twd, ty, a2, GEMM_BN, st)) != SFFN_OK) return r;
    { move_rows_kernel<false><<<g, 256, 0, st>>>(static_cast<const uint4*>(yo), static_cast<uint4*>(Y), list, cnt,
                                               (int)R, (int)(K / 8)); note_launch(); }
    return cudaGetLastError() == cudaSuccess ? SFFN_OK : SFFN_ERR_CUDA;
}

int sffn_twell_to_hybrid(const uint32_t* twell, int64_t M, int64_t N, int T, int C, int ell_w, void* ell_val,
                         int16_t* ell_col, int32_t* row_nnz, int32_t* row_loc, int64_t dense_cap, void* dense_rows,
                         int32_t* dense_map, int* d_dense_count, double* d_l0l1, void* stream) {
    if (!valid_TC(T, C)) return SFFN_ERR_INVALID_ARG;
    if (M < 0 || N <= 0 || N % T != 0 || N > 65536 || ell_w < 1 || dense_cap < 0) return SFFN_ERR_SHAPE;
    if (M == 0) return SFFN_OK;
    if (!twell || !ell_val || !ell_col || !row_nnz || !row_loc || !d_dense_count) return SFFN_ERR_INVALID_ARG;
    if (dense_cap > 0 && (!dense_rows || !dense_map)) return SFFN_ERR_INVALID_ARG;
    int r = check_device();
    if (r != SFFN_OK) return r;
    { twell_to_hybrid_kernel<<<static_cast<unsigned>((M * 32 + 255) / 256), 256, 0, S(stream)>>>(
        twell, (int)M, (int)N, T, C, ell_w, static_cast<uint16_t*>(ell_val), ell_col, row_nnz, row_loc,
        (int)dense_cap, static_cast<uint16_t*>(dense_rows), dense_map, d_dense_count, d_l0l1); note_launch(); }
    return cudaGetLastError() == cudaSuccess ? SFFN_OK : SFFN_ERR_CUDA;
}

// ---------------------------------------------------------------- training forward via the union path (NEXT-4)
int sffn_forward_train(const void* X, const void* Wg, const void* Wu, const void* Wd, int64_t M, int64_t K, int64_t N,
                       int T, int C, void* Y, int ell_w, void* ell_g, void* ell_h, int16_t* ell_col, int32_t* row_nnz,
                       int32_t* row_loc, int64_t dense_cap, void* dense_g, void* dense_h, int32_t* dense_map,
                       int* d_dense_count, double* d_l0l1, void* workspace, size_t ws_bytes, uint32_t* d_overflow,
                       void* stream) {
    if (!union_applicable(N)) return SFFN_ERR_SHAPE;
    if (M > 0 && (!ell_g || !ell_h || (dense_cap > 0 && !dense_h))) return SFFN_ERR_INVALID_ARG;
    int r = sffn_forward(X, Wg, Wu, Wd, M, K, N, T, C, Y, workspace, ws_bytes, d_overflow, SFFN_ALGO_UNION, stream);
    if (r != SFFN_OK || M == 0) return r;
    const uint32_t* tw = static_cast<const uint32_t*>(workspace);
    if ((r = sffn_twell_to_hybrid(tw, M, N, T, C, ell_w, ell_g, ell_col, row_nnz, row_loc, dense_cap, dense_g,
                                  dense_map, d_dense_count, d_l0l1, stream)) != SFFN_OK)
        return r;
    const int64_t tw_bytes = align1k(sffn_twell_words(M, N, T, C) * 4);
    uint8_t* base = static_cast<uint8_t*>(workspace) + tw_bytes;
    UnionWs L = union_ws_layout(M, N, K, T, C);
    { union_h_to_hybrid_kernel<<<static_cast<unsigned>((M * 32 + 255) / 256), 256, 0, S(stream)>>>(
        reinterpret_cast<const uint16_t*>(base + L.hc), (int)M, (int)N, union_brows(),
        reinterpret_cast<const int32_t*>(base + L.perm), reinterpret_cast<const uint32_t*>(base + L.glist),
        reinterpret_cast<const uint16_t*>(base + L.coff), L.lmax, L.nchunk, reinterpret_cast<const int32_t*>(base + L.ulist),
        row_nnz, row_loc, ell_w, static_cast<uint16_t*>(ell_h), static_cast<uint16_t*>(dense_h), tw, T, C,
        reinterpret_cast<const int32_t*>(base + L.udense)); note_launch(); }
    return cudaGetLastError() == cudaSuccess ? SFFN_OK : SFFN_ERR_CUDA;
}

// ---------------------------------------------------------------- training forward on the hybrid format (NEXT-4)
size_t sffn_hybrid_mm_workspace_bytes(int64_t D, int64_t K, int64_t N) {
    if (D < 0 || K <= 0 || N <= 0) return 0;
    const int64_t Dp = ((D + 127) / 128) * 128;
    const int64_t sddmm = align1k(Dp * K * 2) + align1k(Dp * N * 4);
    return static_cast<size_t>(std::max<int64_t>(sddmm, align1k(Dp * K * 2)));
}

int sffn_hybrid_sddmm(const void* A, const void* B, int64_t M, int64_t K, int64_t N, int ell_w, const int16_t* ell_col,
                      const int32_t* row_nnz, const int32_t* row_loc, const void* P_ell, int64_t D,
                      const int32_t* dense_map, const int* d_dense_count, const void* P_dense, int gate, void* out_ell,
                      void* out_dense, void* workspace, size_t ws_bytes, void* stream) {
    if (M < 0 || D < 0 || ell_w < 1 || K < 64 || K % 64 != 0 || N < 16 || N % 16 != 0 || N > 65536)
        return SFFN_ERR_SHAPE;
    if (M == 0) return SFFN_OK;
    if (!A || !B || !ell_col || !row_nnz || !row_loc || !out_ell || (gate && !P_ell)) return SFFN_ERR_INVALID_ARG;
    if (D > 0 && (!dense_map || !d_dense_count || !P_dense || !out_dense || !workspace)) return SFFN_ERR_INVALID_ARG;
    if (!aligned16(A) || !aligned16(B)) return SFFN_ERR_INVALID_ARG;
    if (D > 0 && ws_bytes < sffn_hybrid_mm_workspace_bytes(D, K, N)) return SFFN_ERR_SHAPE;
    if (D > 0 && N < GEMM_BN) return SFFN_ERR_SHAPE;  // the tail GEMM's B box is 256 rows
    int r = check_device();
    if (r != SFFN_OK) return r;
    cudaStream_t st = S(stream);
    { hybrid_sddmm_ell_kernel<<<static_cast<unsigned>(M), HMM_WARPS * 32, 0, st>>>(
        static_cast<const uint4*>(A), static_cast<const uint4*>(B), (int)(K / 8), ell_w, ell_col, row_nnz, row_loc,
        static_cast<const uint16_t*>(P_ell), gate, static_cast<uint16_t*>(out_ell)); note_launch(); }
    if (cudaGetLastError() != cudaSuccess) return SFFN_ERR_CUDA;
    if (D == 0) return SFFN_OK;
    // dense tail: gather the tail rows of A, fp32 tcgen05 GEMM against B, mask (and gate) by the pattern
    const int64_t Dp = ((D + 127) / 128) * 128;
    uint8_t* w = static_cast<uint8_t*>(workspace);
    void* Ad = w;
    float* S32 = reinterpret_cast<float*>(w + align1k(Dp * K * 2));
    const unsigned g = static_cast<unsigned>((Dp * 32 + 255) / 256);
    { move_rows_kernel<true><<<g, 256, 0, st>>>(static_cast<const uint4*>(A), static_cast<uint4*>(Ad), dense_map,
                                              d_dense_count, (int)D, (int)(K / 8)); note_launch(); }
    if (cudaGetLastError() != cudaSuccess) return SFFN_ERR_CUDA;
    CUtensorMap ta, tb;
    if (!tmap_2d(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Ad, K, Dp, GEMM_BK, GEMM_BM, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !tmap_2d(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, B, K, N, GEMM_BK, GEMM_BN, CU_TENSOR_MAP_SWIZZLE_128B))
        return SFFN_ERR_CUDA;
    GemmArgs ga{};
    ga.M = (int)Dp;
    ga.N = (int)N;
    ga.K = (int)K;
    ga.out_f32 = S32;
    ga.ld_out = N;
    ga.m_dev = d_dense_count;
    if ((r = launch_gemm<EPI_F32, 1>(ta, tb, tb, tb, ga, GEMM_BN, st)) != SFFN_OK) return r;
    { hybrid_tail_mask_kernel<<<dev_info().sms * 4, 256, 0, st>>>(S32, static_cast<const uint16_t*>(P_dense), N,
                                                                 d_dense_count, (int)D, gate,
                                                                 static_cast<uint16_t*>(out_dense)); note_launch(); }
    return cudaGetLastError() == cudaSuccess ? SFFN_OK : SFFN_ERR_CUDA;
}

int sffn_hybrid_spmm(const void* ell_val, const int16_t* ell_col, const int32_t* row_nnz, const int32_t* row_loc,
                     int64_t M, int ell_w, int64_t D, const int32_t* dense_map, const int* d_dense_count,
                     const void* dense, const void* W, int64_t N, int64_t K, void* Y, void* workspace, size_t ws_bytes,
                     void* stream) {
    if (M < 0 || D < 0 || ell_w < 1 || K < 256 || K % 64 != 0 || N < 64 || N % 64 != 0 || N > 65536)
        return SFFN_ERR_SHAPE;
    if (M == 0) return SFFN_OK;
    if (!ell_val || !ell_col || !row_nnz || !row_loc || !W || !Y) return SFFN_ERR_INVALID_ARG;
    if (D > 0 && (!dense_map || !d_dense_count || !dense || !workspace)) return SFFN_ERR_INVALID_ARG;
    if (!aligned16(W) || !aligned16(Y)) return SFFN_ERR_INVALID_ARG;
    if (D > 0 && ws_bytes < sffn_hybrid_mm_workspace_bytes(D, K, N)) return SFFN_ERR_SHAPE;
    int r = check_device();
    if (r != SFFN_OK) return r;
    cudaStream_t st = S(stream);
    { hybrid_spmm_ell_kernel<<<static_cast<unsigned>(M), 128, 0, st>>>(
        static_cast<const uint16_t*>(ell_val), ell_col, row_nnz, row_loc, ell_w, static_cast<const uint4*>(W),
        (int)(K / 8), static_cast<uint4*>(Y)); note_launch(); }
    if (cudaGetLastError() != cudaSuccess) return SFFN_ERR_CUDA;
    if (D == 0) return SFFN_OK;
    // dense tail: tcgen05 GEMM of the tail rows with W (read MN-major by TMA), rows scattered to Y[dense_map[s]]
    const int64_t Dp = ((D + 127) / 128) * 128;
    void* Yd = workspace;
    CUtensorMap th, tw, ty;
    if (!tmap_2d(&th, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dense, N, D, GEMM_BK, GEMM_BM, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !tmap_2d(&tw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, W, K, N, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !tmap_2d(&ty, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Yd, K, Dp, 128, 32, CU_TENSOR_MAP_SWIZZLE_NONE))
        return SFFN_ERR_CUDA;
    GemmArgs ga{};
    ga.M = (int)Dp;
    ga.N = (int)K;
    ga.K = (int)N;
    ga.m_dev = d_dense_count;
    if ((r = launch_gemm<EPI_BF16_MN, 1>(th, tw, tw, ty, ga, GEMM_BN, st)) != SFFN_OK) return r;
    const unsigned g = static_cast<unsigned>((Dp * 32 + 255) / 256);
    { move_rows_kernel<false><<<g, 256, 0, st>>>(static_cast<const uint4*>(Yd), static_cast<uint4*>(Y), dense_map,
                                               d_dense_count, (int)D, (int)(K / 8)); note_launch(); }
    return cudaGetLastError() == cudaSuccess ? SFFN_OK : SFFN_ERR_CUDA;
}

int sffn_union_block_rows(void) { return union_brows(); }

int sffn_union_stats(const void* workspace, int64_t M, int64_t K, int64_t N, int64_t* padded_sum, int64_t* real_sum,
                     int64_t* up_tiles, void* stream) {
    if (!workspace || M <= 0 || N <= 0 || K <= 0) return SFFN_ERR_INVALID_ARG;
    const int64_t NB = (M + union_brows() - 1) / union_brows();
    UnionWs L = union_ws_layout(M, N, K);
    const uint8_t* base = static_cast<const uint8_t*>(workspace);
    int32_t* h = static_cast<int32_t*>(std::malloc(static_cast<size_t>(2 * NB + 1) * 4));
    if (!h) return SFFN_ERR_INVALID_ARG;
    cudaStream_t st = S(stream);
    int r = SFFN_OK;
    if (cudaMemcpyAsync(h, base + L.ulen, NB * 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaMemcpyAsync(h + NB, base + L.utot, NB * 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaMemcpyAsync(h + 2 * NB, base + L.chunk, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        r = SFFN_ERR_CUDA;
    if (r == SFFN_OK) {
        int64_t a = 0, b = 0;
        for (int64_t i = 0; i < NB; ++i) {
            a += h[i];
            b += h[NB + i];
        }
        if (padded_sum) *padded_sum = a;
        if (real_sum) *real_sum = b;
        if (up_tiles) *up_tiles = h[2 * NB];
    }
    std::free(h);
    return r;
}

int sffn_overflow_check(const uint32_t* d_overflow, void* stream, uint32_t* host_count) {
    if (!d_overflow) return SFFN_ERR_INVALID_ARG;
    uint32_t h = 0;
    if (cudaMemcpyAsync(&h, d_overflow, 4, cudaMemcpyDeviceToHost, S(stream)) != cudaSuccess) return SFFN_ERR_CUDA;
    if (cudaStreamSynchronize(S(stream)) != cudaSuccess) return SFFN_ERR_CUDA;
    if (host_count) *host_count = h;
    return h ? SFFN_ERR_TILE_OVERFLOW : SFFN_OK;
}

}  // extern "C"
