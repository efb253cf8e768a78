// Streaming ceiling on this B200 for the fused step's access pattern:
// 3 read streams + 3 write streams (float4, grid-stride), against a 1:1 copy.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/hbm_probe tools/hbm_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void r3w3(const float4* __restrict__ a, const float4* __restrict__ b, const float4* __restrict__ c,
                     float4* __restrict__ d, float4* __restrict__ e, float4* __restrict__ f, long n) {
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
        float4 x = __ldcs(a + i), y = __ldcs(b + i), z = __ldcs(c + i);
        float4 m = make_float4(0.9f * z.x + y.x, 0.9f * z.y + y.y, 0.9f * z.z + y.z, 0.9f * z.w + y.w);
        float4 w = make_float4(x.x - 0.1f * m.x, x.y - 0.1f * m.y, x.z - 0.1f * m.z, x.w - 0.1f * m.w);
        __stcs(d + i, m);
        __stcs(e + i, w);
        __stcs(f + i, w);
    }
}
__global__ void copy1(const float4* __restrict__ a, float4* __restrict__ d, long n) {
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x)
        __stcs(d + i, __ldcs(a + i));
}

int main() {
    const long n = 200l << 20;  // float4 elements per stream: 3.2 GB per stream
    float4* p[6];
    for (int i = 0; i < 6; ++i) {
        if (cudaMalloc(&p[i], n * 16) != cudaSuccess) { printf("oom\n"); return 1; }
        cudaMemset(p[i], 0, n * 16);
    }
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int per : {4, 8, 16}) {
        for (int bs : {256, 512}) {
            float best = 1e9f, bestc = 1e9f;
            for (int it = 0; it < 6; ++it) {
                cudaEventRecord(e0);
                r3w3<<<sms * per, bs>>>(p[0], p[1], p[2], p[3], p[4], p[5], n / 4);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (it) best = ms < best ? ms : best;
                cudaEventRecord(e0);
                copy1<<<sms * per, bs>>>(p[0], p[3], n);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
                if (it) bestc = ms < bestc ? ms : bestc;
            }
            printf("ctas/SM %2d block %3d: r3w3 %.1f GB/s   copy %.1f GB/s\n", per, bs,
                   6.0 * (n / 4) * 16 / (best * 1e6), 2.0 * n * 16 / (bestc * 1e6));
        }
    }
    return 0;
}
