// Experiment: semantics of cp.async.bulk.tensor.2d ... tile::gather4 on sm_100a.
//  - which tensor-map box[1] is accepted (1 or 4)
//  - where the 4 rows land in shared memory, and whether the 128B swizzle is address-based
//    (issue a gather4 at +512 B inside a 1024-B aligned atom).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o tools/exp_gather4 tools/exp_gather4.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../paper_2603_23198_b200/csrc/ptx.cuh"

using namespace sffn;

__global__ void k_gather(const __grid_constant__ CUtensorMap tm, uint16_t* out, int mode) {
    __shared__ __align__(1024) uint8_t buf[2048];
    __shared__ uint64_t bar;
    for (int i = threadIdx.x; i < 2048 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(buf)[i] = 0xFFFFFFFFu;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bar, 1024);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(buf)),
            "l"(reinterpret_cast<uint64_t>(&tm)), "r"(smem_u32(&bar)), "r"(64), "r"(5), "r"(17), "r"(2), "r"(40)
            : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(buf + 512)),
            "l"(reinterpret_cast<uint64_t>(&tm)), "r"(smem_u32(&bar)), "r"(128), "r"(7), "r"(8), "r"(9), "r"(10)
            : "memory");
        mbar_wait(&bar, 0);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 1024 / 2; i += blockDim.x) out[i] = reinterpret_cast<uint16_t*>(buf)[i];
}

typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const int R = 64, Ccols = 256;
    std::vector<uint16_t> h(R * Ccols);
    for (int r = 0; r < R; ++r)
        for (int c = 0; c < Ccols; ++c) h[r * Ccols + c] = (uint16_t)(r * 256 + c);  // row in high byte, col low
    uint16_t *d, *o;
    cudaMalloc(&d, h.size() * 2);
    cudaMalloc(&o, 1024);
    cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
    void* p;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    PFN enc = (PFN)p;
    for (int box1 : {1, 4}) {
        CUtensorMap tm;
        cuuint64_t dims[2] = {(cuuint64_t)Ccols, (cuuint64_t)R};
        cuuint64_t str[1] = {(cuuint64_t)Ccols * 2};
        cuuint32_t box[2] = {64, (cuuint32_t)box1};
        cuuint32_t es[2] = {1, 1};
        CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("box1=%d encode=%d\n", box1, (int)r);
        if (r != CUDA_SUCCESS) continue;
        cudaMemset(o, 0, 1024);
        k_gather<<<1, 128>>>(tm, o, 0);
        cudaError_t e = cudaDeviceSynchronize();
        printf("  kernel: %s\n", cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
        std::vector<uint16_t> out(512);
        cudaMemcpy(out.data(), o, 1024, cudaMemcpyDeviceToHost);
        // print, per 128-B smem row, the (row, col) of the first element of each 16-B chunk
        for (int sr = 0; sr < 8; ++sr) {
            printf("  smem row %d:", sr);
            for (int ch = 0; ch < 8; ++ch) {
                uint16_t v = out[sr * 64 + ch * 8];
                printf(" (%d,%d)", v >> 8, v & 255);
            }
            printf("\n");
        }
    }
    return 0;
}
