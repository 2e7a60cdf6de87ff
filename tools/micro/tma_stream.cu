// TMA streaming bandwidth per box shape (the seed's access pattern): every
// CTA (one per SM) streams its share of a [rows][256] fp32 matrix through a
// ring of shared-memory slots, consumers touch one word per slot, and the
// achieved GB/s is printed per box shape.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_stream tma_stream.cu -lcuda && ./tma_stream
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbi(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c)); }
__device__ __forceinline__ void mbtx(uint64_t* b, uint32_t x) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(x) : "memory"); }
__device__ __forceinline__ void mba(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory"); }
__device__ __forceinline__ void mbw(uint64_t* b, uint32_t ph) {
    asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}" ::"r"(su(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma(void* d, const CUtensorMap* m, int x, int y, uint64_t* b) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(su(d)), "l"((uint64_t)m), "r"(x), "r"(y), "r"(su(b)) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su(d)), "l"(s), "r"(n), "r"(su(b)) : "memory");
}

// box (bw dims x bh rows), slot = nbx boxes along rows; walk: for each row block of 1024 rows,
// for each dim window of bw, the 1024 rows (like the seed's slices)
__global__ void stream_kernel(const __grid_constant__ CUtensorMap m, const float* base, int rows, int dim, int bw, int bh,
                              int stages, int mode, float* sink) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* ring = sm + 1024;
    uint64_t* full = (uint64_t*)sm;
    uint64_t* empty = full + 32;
    const int slot_bytes = 1024 * bw * 4;  // 1024 rows x bw dims
    if (threadIdx.x == 0) {
        for (int i = 0; i < stages; ++i) { mbi(full + i, 1); mbi(empty + i, (blockDim.x / 32) - 1); }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const int groups = rows / 1024;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int nwin = dim / bw;
    if (warp == 0) {
        if (lane) return;
        int sl = 0;
        for (int g = blockIdx.x; g < groups; g += gridDim.x)
            for (int k = 0; k < nwin; ++k, ++sl) {
                const int s = sl % stages;
                if (sl >= stages) mbw(empty + s, ((sl / stages) - 1) & 1);
                mbtx(full + s, slot_bytes);
                if (mode == 0) {
                    for (int r = 0; r < 1024; r += bh) tma(ring + s * slot_bytes + r * bw * 4, &m, k * bw, g * 1024 + r, full + s);
                } else {  // mode 1: contiguous 1D bulk copies of whole rows (bw == dim)
                    bulk(ring + s * slot_bytes, base + (size_t)g * 1024 * dim + (size_t)k * 0, slot_bytes, full + s);
                }
            }
        return;
    }
    float acc = 0.f;
    int sl = 0;
    for (int g = blockIdx.x; g < groups; g += gridDim.x)
        for (int k = 0; k < nwin; ++k, ++sl) {
            const int s = sl % stages;
            mbw(full + s, (sl / stages) & 1);
            acc += ((float*)(ring + s * slot_bytes))[threadIdx.x];
            __syncwarp();
            if (lane == 0) mba(empty + s);
        }
    if (acc == 12345.f) sink[0] = acc;
}

int main() {
    const int dim = 256;
    const size_t rows = 1 << 20;
    float* d;
    cudaMalloc(&d, rows * dim * 4);
    cudaMemset(d, 0, rows * dim * 4);
    float* sink;
    cudaMalloc(&sink, 4);
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    struct Cfg { int bw, bh, swz, promo, stages_bytes; };
    std::vector<Cfg> cfgs = {{8, 256, 1, 256, 128}, {8, 256, 1, 256, 192}, {16, 256, 2, 256, 128}, {32, 256, 3, 256, 128},
                             {32, 128, 3, 256, 128}, {8, 256, 1, 128, 128}, {8, 256, 1, 0, 128}, {32, 256, 3, 256, 192}};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (auto c : cfgs) {
        CUtensorMap m;
        cuuint64_t gd[2] = {(cuuint64_t)dim, (cuuint64_t)rows};
        cuuint64_t gs[1] = {(cuuint64_t)dim * 4};
        cuuint32_t box[2] = {(cuuint32_t)c.bw, (cuuint32_t)c.bh};
        cuuint32_t es[2] = {1, 1};
        CUtensorMapSwizzle sw = c.swz == 1 ? CU_TENSOR_MAP_SWIZZLE_32B : c.swz == 2 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
        CUtensorMapL2promotion pr = c.promo == 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : c.promo == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE;
        if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, pr,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("encode failed\n"); continue; }
        const int slot_bytes = 1024 * c.bw * 4;
        const int stages = (c.stages_bytes * 1024) / slot_bytes;
        const int smem = 1024 + stages * slot_bytes;
        cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        for (int it = 0; it < 2; ++it) stream_kernel<<<nsm, 288, smem>>>(m, d, (int)rows, dim, c.bw, c.bh, stages, 0, sink);
        cudaEventRecord(e0);
        stream_kernel<<<nsm, 288, smem>>>(m, d, (int)rows, dim, c.bw, c.bh, stages, 0, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("box {%d dims, %d rows} swz %d promo %d ring %d KB (%d stages): %.1f us, %.0f GB/s  %s\n", c.bw, c.bh, c.swz, c.promo,
               stages * slot_bytes / 1024, stages, ms * 1e3, rows * dim * 4 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
