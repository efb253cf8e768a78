// NVLink pull microbenchmark: how fast can one GPU read a peer GPU's memory?
//   mode 0: 128-bit LDG (ld.global.cg) by every thread
//   mode 1: TMA bulk copies (cp.async.bulk global->shared, mbarrier) issued by one thread per CTA
//   mode 2: cp.async (LDGSTS) 16 B per thread into a per-thread ring
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvl_probe tools/nvl_probe.cu
// Run on a box with >= 2 GPUs: tools/nvl_probe [bytes]
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void ldg_kernel(const float4* __restrict__ src, size_t n16, float* out) {
    float acc = 0.f;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x) {
        float4 v = __ldcg(src + i);
        acc += v.x + v.y + v.z + v.w;
    }
    if (acc == 1234.5f) out[0] = acc;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
            (unsigned)__cvta_generic_to_shared(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
                 : "memory");
}

constexpr int kStages = 4;
constexpr int kChunk = 16384;  // bytes per stage

__global__ void tma_kernel(const char* src, size_t bytes, float* out) {
    extern __shared__ __align__(128) char smem[];
    __shared__ uint64_t bars[kStages];
    const size_t nchunks = bytes / kChunk;
    if (threadIdx.x == 0)
        for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    size_t c0 = blockIdx.x;
    // prologue
    if (threadIdx.x == 0)
        for (int s = 0; s < kStages; ++s) {
            size_t c = c0 + size_t(s) * gridDim.x;
            if (c < nchunks) {
                mbar_expect_tx(&bars[s], kChunk);
                bulk_g2s(smem + s * kChunk, src + c * kChunk, kChunk, &bars[s]);
            }
        }
    float acc = 0.f;
    int it = 0;
    for (size_t c = c0; c < nchunks; c += gridDim.x, ++it) {
        const int s = it % kStages;
        mbar_wait(&bars[s], (it / kStages) & 1);
        const float4* v = reinterpret_cast<const float4*>(smem + s * kChunk);
        for (int i = threadIdx.x; i < kChunk / 16; i += blockDim.x) {
            float4 x = v[i];
            acc += x.x + x.y + x.z + x.w;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            size_t cn = c + size_t(kStages) * gridDim.x;
            if (cn < nchunks) {
                mbar_expect_tx(&bars[s], kChunk);
                bulk_g2s(smem + s * kChunk, src + cn * kChunk, kChunk, &bars[s]);
            }
        }
    }
    if (acc == 1234.5f) out[0] = acc;
}

// all-to-all: chunk c comes from source c % nsrc (every peer read concurrently)
struct Srcs { const char* p[8]; };
__global__ void tma_multi_kernel(Srcs srcs, int nsrc, size_t bytes_per_src, float* out) {
    extern __shared__ __align__(128) char smem[];
    __shared__ uint64_t bars[kStages];
    const size_t per = bytes_per_src / kChunk, nchunks = per * nsrc;
    if (threadIdx.x == 0)
        for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    auto src_of = [&](size_t c) { return srcs.p[c % nsrc] + (c / nsrc) * kChunk; };
    if (threadIdx.x == 0)
        for (int s = 0; s < kStages; ++s) {
            size_t c = blockIdx.x + size_t(s) * gridDim.x;
            if (c < nchunks) {
                mbar_expect_tx(&bars[s], kChunk);
                bulk_g2s(smem + s * kChunk, src_of(c), kChunk, &bars[s]);
            }
        }
    float acc = 0.f;
    int it = 0;
    for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
        const int s = it % kStages;
        mbar_wait(&bars[s], (it / kStages) & 1);
        const float4* v = reinterpret_cast<const float4*>(smem + s * kChunk);
        for (int i = threadIdx.x; i < kChunk / 16; i += blockDim.x) {
            float4 x = v[i];
            acc += x.x + x.y + x.z + x.w;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            size_t cn = c + size_t(kStages) * gridDim.x;
            if (cn < nchunks) {
                mbar_expect_tx(&bars[s], kChunk);
                bulk_g2s(smem + s * kChunk, src_of(cn), kChunk, &bars[s]);
            }
        }
    }
    if (acc == 1234.5f) out[0] = acc;
}

// all-to-all push: every thread stores 16-B vectors into the peers' buffers
struct Dsts { float4* p[8]; };
__global__ void push_multi_kernel(Dsts dsts, int ndst, size_t n16_per_dst) {
    const size_t total = n16_per_dst * ndst;
    const float4 v = make_float4(1.f, 2.f, 3.f, float(threadIdx.x));
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total; i += size_t(gridDim.x) * blockDim.x) {
        const size_t chunk = i / 1024;  // 16 KB chunks round-robin over the peers
        dsts.p[chunk % ndst][(chunk / ndst) * 1024 + (i % 1024)] = v;
    }
}

// HBM streaming copy, to load the memory system while the pulls run
__global__ void hbm_copy_kernel(const float4* a, float4* b, size_t n16) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x)
        b[i] = __ldcs(a + i);
}

static int all_to_all(int n, size_t bytes, bool with_hbm) {
    // every GPU pulls `bytes` from each of its n-1 peers at the same time
    char* buf[8];
    float* out[8];
    float4 *ha[8], *hb[8];
    const size_t hbm_bytes = size_t(2) << 30;
    for (int g = 0; g < n; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaMalloc(&buf[g], bytes));
        CK(cudaMemset(buf[g], 0, bytes));
        CK(cudaMalloc(&out[g], 4));
        CK(cudaMalloc(&ha[g], hbm_bytes));
        CK(cudaMalloc(&hb[g], hbm_bytes));
        for (int q = 0; q < n; ++q)
            if (q != g) {
                cudaError_t pe = cudaDeviceEnablePeerAccess(q, 0);
                if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) CK(pe);
                cudaGetLastError();
            }
        CK(cudaFuncSetAttribute(tma_multi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kChunk));
    }
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t a[8], b[8], c[8], d[8];
    cudaStream_t s1[8], s2[8];
    for (int g = 0; g < n; ++g) {
        CK(cudaSetDevice(g));
        cudaEventCreate(&a[g]); cudaEventCreate(&b[g]); cudaEventCreate(&c[g]); cudaEventCreate(&d[g]);
        cudaStreamCreateWithFlags(&s1[g], cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&s2[g], cudaStreamNonBlocking);
    }
    // push: every GPU writes `bytes` into each peer at once
    for (int rep = 0; rep < 3; ++rep) {
        for (int g = 0; g < n; ++g) {
            CK(cudaSetDevice(g));
            Dsts dsts;
            int k = 0;
            for (int q = 0; q < n; ++q)
                if (q != g) dsts.p[k++] = reinterpret_cast<float4*>(buf[q]);
            cudaEventRecord(a[g], s1[g]);
            push_multi_kernel<<<sms * 4, 256, 0, s1[g]>>>(dsts, n - 1, bytes / 16 / n);
            cudaEventRecord(b[g], s1[g]);
        }
        for (int g = 0; g < n; ++g) {
            CK(cudaSetDevice(g));
            CK(cudaDeviceSynchronize());
            CK(cudaGetLastError());
            float ms;
            cudaEventElapsedTime(&ms, a[g], b[g]);
            if (rep == 2 && !with_hbm)
                printf("a2a push n=%d gpu %d: %.3f ms %.1f GB/s egress\n", n, g, ms, (bytes / n) * (n - 1) / ms / 1e6);
        }
    }
    for (int rep = 0; rep < 3; ++rep) {
        for (int g = 0; g < n; ++g) {
            CK(cudaSetDevice(g));
            Srcs srcs;
            int k = 0;
            for (int q = 0; q < n; ++q)
                if (q != g) srcs.p[k++] = buf[q];
            const int pull_ctas = with_hbm ? sms / 2 : sms;
            cudaEventRecord(a[g], s1[g]);
            tma_multi_kernel<<<pull_ctas, 128, kStages * kChunk, s1[g]>>>(srcs, n - 1, bytes, out[g]);
            cudaEventRecord(b[g], s1[g]);
            if (with_hbm) {
                cudaEventRecord(c[g], s2[g]);
                hbm_copy_kernel<<<sms * 4, 256, 0, s2[g]>>>(ha[g], hb[g], hbm_bytes / 16);
                cudaEventRecord(d[g], s2[g]);
            }
        }
        for (int g = 0; g < n; ++g) {
            CK(cudaSetDevice(g));
            CK(cudaDeviceSynchronize());
            CK(cudaGetLastError());
            float ms, ms2 = 0.f;
            cudaEventElapsedTime(&ms, a[g], b[g]);
            if (with_hbm) cudaEventElapsedTime(&ms2, c[g], d[g]);
            if (rep == 2)
                printf("a2a n=%d gpu %d: pull %.3f ms %.1f GB/s ingress%s", n, g, ms, bytes * (n - 1) / ms / 1e6,
                       with_hbm ? "" : "\n");
            if (rep == 2 && with_hbm) printf("  | hbm copy %.3f ms %.1f GB/s\n", ms2, 2.0 * hbm_bytes / ms2 / 1e6);
        }
    }
    for (int g = 0; g < n; ++g) {
        CK(cudaSetDevice(g));
        cudaFree(buf[g]); cudaFree(out[g]); cudaFree(ha[g]); cudaFree(hb[g]);
    }
    return 0;
}

__global__ void cpasync_kernel(const float4* src, size_t n16, float* out) {
    extern __shared__ __align__(16) float4 ring[];  // [4][blockDim]
    float acc = 0.f;
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    size_t i0 = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    constexpr int D = 4;
    for (int d = 0; d < D; ++d) {
        size_t i = i0 + d * stride;
        if (i < n16) {
            unsigned s = (unsigned)__cvta_generic_to_shared(&ring[d * blockDim.x + threadIdx.x]);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(src + i) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    int k = 0;
    for (size_t i = i0; i < n16; i += stride, ++k) {
        asm volatile("cp.async.wait_group 3;" ::: "memory");
        float4 x = ring[(k % D) * blockDim.x + threadIdx.x];
        acc += x.x + x.y + x.z + x.w;
        size_t nx = i + D * stride;
        if (nx < n16) {
            unsigned s = (unsigned)__cvta_generic_to_shared(&ring[(k % D) * blockDim.x + threadIdx.x]);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(src + nx) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    if (acc == 1234.5f) out[0] = acc;
}

int main(int argc, char** argv) {
    size_t bytes = argc > 1 ? strtoull(argv[1], nullptr, 10) : (size_t(1) << 30);
    int n;
    CK(cudaGetDeviceCount(&n));
    if (argc > 2 && argv[2][0] == 'a') {  // tools/nvl_probe BYTES a2a: all-to-all pulls
        for (int k = 2; k <= n; k *= 2) {
            if (all_to_all(k, bytes / 4, false)) return 1;
            if (all_to_all(k, bytes / 4, true)) return 1;
        }
        return 0;
    }
    int peer = n > 1 ? 1 : 0;
    char* buf;
    CK(cudaSetDevice(peer));
    CK(cudaMalloc(&buf, bytes));
    CK(cudaMemset(buf, 0, bytes));
    CK(cudaSetDevice(0));
    if (peer) CK(cudaDeviceEnablePeerAccess(peer, 0));
    float* out;
    CK(cudaMalloc(&out, 4));
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kChunk));
    CK(cudaFuncSetAttribute(cpasync_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 1024 * 16));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    printf("reading %zu bytes of GPU %d memory from GPU 0 (%s)\n", bytes, peer, peer ? "NVLink" : "local HBM");
    for (int mode = 0; mode < 3; ++mode) {
        for (int cfg = 0; cfg < 3; ++cfg) {
            int per_sm = cfg == 0 ? 1 : (cfg == 1 ? 2 : 4);
            int threads = 256;
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(a);
                if (mode == 0) ldg_kernel<<<sms * per_sm * 2, threads>>>((const float4*)buf, bytes / 16, out);
                if (mode == 1) tma_kernel<<<sms * per_sm, 128, kStages * kChunk>>>(buf, bytes, out);
                if (mode == 2) cpasync_kernel<<<sms * per_sm, threads, 4 * threads * 16>>>((const float4*)buf, bytes / 16, out);
                cudaEventRecord(b);
                CK(cudaEventSynchronize(b));
                CK(cudaGetLastError());
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (rep == 2)
                    printf("mode %d (%s) ctas/sm=%d: %.3f ms  %.1f GB/s\n", mode,
                           mode == 0 ? "ldg.cg" : (mode == 1 ? "tma bulk" : "cp.async"), per_sm * (mode == 0 ? 2 : 1), ms,
                           bytes / ms / 1e6);
            }
        }
    }
    return 0;
}
