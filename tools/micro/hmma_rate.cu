// Microbenchmark: legacy mma.sync m16n8k8 TF32 issue rate on this GPU
// (nvcc -gencode arch=compute_100a,code=sm_100a -O3 hmma_rate.cu -o hmma_rate)
#include <cstdio>
#include <cstdint>
__global__ void k(float* out, int iters) {
    float d[8][4] = {};
    uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                         : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
    for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    float* out; cudaMalloc(&out, 148 * 32 * 1024 * 4);
    int iters = 4096;
    for (int warps : {4, 8, 16, 32}) {
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        k<<<148, warps * 32>>>(out, 16);
        cudaEventRecord(e0);
        k<<<148, warps * 32>>>(out, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double hmma = 148.0 * warps * iters * 8;
        printf("warps/SM %2d: %.3f ms  %.2f HMMA/cycle/SM (at 1.965 GHz)  %.1f TFLOP/s tf32\n", warps, ms,
               hmma / (ms * 1e-3) / 148 / 1.965e9, hmma * 16 * 8 * 8 * 2 / (ms * 1e-3) / 1e12);
    }
    return 0;
}
