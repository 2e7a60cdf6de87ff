// Host->device transfer paths for a pinned 10 MiB query block (diagnostic):
// one DMA copy, the copy split over several streams (copy engines), and SM loads
// of the mapped pinned buffer (zero-copy) into device memory; plus the D2H analogues.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a h2d_paths.cu -o h2d_paths
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void pull_kernel(const float4* __restrict__ src, float4* __restrict__ dst, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        dst[i] = src[i];
    }
}
__global__ void pull_kernel_u(const float4* __restrict__ src, float4* __restrict__ dst, size_t n) {
    // 4 independent loads in flight per thread
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n; i += 4 * stride) {
        float4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
        dst[i] = a; dst[i + stride] = b; dst[i + 2 * stride] = c; dst[i + 3 * stride] = d;
    }
    for (; i < n; i += stride) dst[i] = src[i];
}

__global__ void spin_kernel(float* out, int iters) {
    float a = threadIdx.x, b = 1.0001f;
    for (int i = 0; i < iters; ++i) a = fmaf(a, b, 0.5f);
    if (a == 12345.f) out[0] = a;
}
__global__ void stream_kernel(const float4* __restrict__ src, float4* __restrict__ dst, size_t n, int reps) {
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
            dst[i] = src[i];
}

int main() {
    const size_t bytes = 10u << 20, n4 = bytes / 16;
    float *h, *d, *d2;
    CK(cudaHostAlloc(&h, bytes, cudaHostAllocDefault));
    for (size_t i = 0; i < bytes / 4; ++i) h[i] = (float)i;
    CK(cudaMalloc(&d, bytes));
    CK(cudaMalloc(&d2, bytes));
    cudaStream_t st[8];
    for (auto& s : st) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
    auto run = [&](const char* name, auto&& body) {
        std::vector<float> ts;
        for (int it = 0; it < 25; ++it) {
            cudaDeviceSynchronize();
            cudaEventRecord(a, st[0]);
            body();
            for (int k = 1; k < 8; ++k) { cudaEvent_t e; cudaEventCreateWithFlags(&e, cudaEventDisableTiming); cudaEventRecord(e, st[k]); cudaStreamWaitEvent(st[0], e, 0); cudaEventDestroy(e); }
            cudaEventRecord(b, st[0]);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (it >= 3) ts.push_back(ms);
        }
        std::sort(ts.begin(), ts.end());
        printf("%-28s min %.3f ms  med %.3f ms  -> %.1f GB/s\n", name, ts[0], ts[ts.size() / 2], bytes / (ts[ts.size() / 2] * 1e6));
    };
    auto fork = [&]() { cudaEvent_t e; cudaEventCreateWithFlags(&e, cudaEventDisableTiming); cudaEventRecord(e, st[0]); for (int k = 1; k < 8; ++k) cudaStreamWaitEvent(st[k], e, 0); cudaEventDestroy(e); };
    run("H2D memcpy x1", [&] { cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st[0]); });
    for (int ns : {2, 4, 8}) {
        char nm[64]; snprintf(nm, sizeof nm, "H2D memcpy split x%d", ns);
        run(nm, [&] { fork(); for (int k = 0; k < ns; ++k) cudaMemcpyAsync((char*)d + bytes / ns * k, (char*)h + bytes / ns * k, bytes / ns, cudaMemcpyHostToDevice, st[k]); });
    }
    for (int blocks : {148, 296, 592, 1184}) {
        char nm[64]; snprintf(nm, sizeof nm, "H2D zero-copy %d blk", blocks);
        run(nm, [&] { pull_kernel<<<blocks, 256, 0, st[0]>>>((const float4*)h, (float4*)d, n4); });
        snprintf(nm, sizeof nm, "H2D zero-copy u4 %d blk", blocks);
        run(nm, [&] { pull_kernel_u<<<blocks, 256, 0, st[0]>>>((const float4*)h, (float4*)d, n4); });
    }
    run("D2H memcpy x1", [&] { cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, st[0]); });
    run("D2H memcpy split x4", [&] { fork(); for (int k = 0; k < 4; ++k) cudaMemcpyAsync((char*)h + bytes / 4 * k, (char*)d + bytes / 4 * k, bytes / 4, cudaMemcpyDeviceToHost, st[k]); });
    run("D2H zero-copy 592 blk", [&] { pull_kernel<<<592, 256, 0, st[0]>>>((const float4*)d, (float4*)h, n4); });
    // H2D while the SMs are busy: FMA-only kernel, and an HBM-streaming kernel
    {
        float* big_a; float* big_b;
        const size_t nb = 256u << 20;
        CK(cudaMalloc(&big_a, nb)); CK(cudaMalloc(&big_b, nb));
        cudaStream_t cs; CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        for (int mode = 0; mode < 2; ++mode) {
            std::vector<float> ts;
            for (int it = 0; it < 12; ++it) {
                cudaDeviceSynchronize();
                if (mode == 0) spin_kernel<<<148 * 8, 256, 0, cs>>>(d2, 200000);
                else stream_kernel<<<148 * 4, 512, 0, cs>>>((const float4*)big_a, (float4*)big_b, nb / 16, 20);
                cudaEventRecord(a, st[0]);
                cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st[0]);
                cudaEventRecord(b, st[0]);
                cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                if (it >= 2) ts.push_back(ms);
                cudaDeviceSynchronize();
            }
            std::sort(ts.begin(), ts.end());
            printf("H2D memcpy during %-12s med %.3f ms -> %.1f GB/s\n", mode ? "HBM stream" : "FMA spin", ts[ts.size() / 2], bytes / (ts[ts.size() / 2] * 1e6));
        }
    }
    // check the zero-copy result
    pull_kernel_u<<<592, 256>>>((const float4*)h, (float4*)d2, n4);
    CK(cudaDeviceSynchronize());
    std::vector<float> back(bytes / 4);
    cudaMemcpy(back.data(), d2, bytes, cudaMemcpyDeviceToHost);
    size_t bad = 0; for (size_t i = 0; i < back.size(); ++i) bad += back[i] != (float)i;
    printf("zero-copy check: %zu mismatches\n", bad);
    return 0;
}
