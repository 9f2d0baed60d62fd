// Microbenchmark (diagnostic, not part of libslim): tcgen05.mma throughput per SM for one CTA
// (cta_group::1, M = 128) vs a CTA pair (cta_group::2, M = 256, the even CTA issuing), same
// per-SM work: n_iter x 12 MMAs (3 A row offsets x 4 K-steps) of N columns into one accumulator.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pair_mma pair_mma.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t a) {
    return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t par) {
    uint32_t ok;
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}" : "=r"(ok) : "r"(bar), "r"(par) : "memory");
    return ok;
}
__device__ __forceinline__ uint32_t elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n .reg .b32 r;\n .reg .pred p;\n elect.sync r|p, 0xffffffff;\n selp.u32 %0, 1, 0, p;\n}" : "=r"(pred));
    return pred;
}
template <int PAIR>
__global__ void mma_rate(int n_iter, int N, int commit_every_kh, unsigned long long *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *s = (uint8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar, dummy;
    __shared__ uint32_t tslot;
    uint32_t rank = 0;
    if (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    if (threadIdx.x < 32) {
        if (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1000000;" ::"r"(smem_u32(&dummy)));   // never completes
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tslot;
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)((PAIR ? 256 : 128) >> 4) << 24);
    const uint64_t ad = desc_sw128(smem_u32(s)), bd = desc_sw128(smem_u32(s + 65536));
    unsigned long long t0 = clock64();
    if (threadIdx.x < 32 && rank == 0) {
        for (int it = 0; it < n_iter; ++it) {
            if (elect_one()) {
#pragma unroll
                for (int kh = 0; kh < 3; ++kh) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint32_t acc = (it | kh | kk) != 0;
                        if (PAIR)
                            asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tm), "l"(ad + kh * 256 + 2 * kk), "l"(bd + 2 * kk), "r"(idesc), "r"(acc));
                        else
                            asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tm), "l"(ad + kh * 256 + 2 * kk), "l"(bd + 2 * kk), "r"(idesc), "r"(acc));
                    }
                    if (commit_every_kh) {   // a per-stage release, as a streamed-weight ring does
                        if (PAIR) asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(&dummy)), "h"((uint16_t)3));
                        else asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&dummy)));
                    }
                }
            }
            __syncwarp();
        }
        if (elect_one()) {
            if (PAIR) asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "h"((uint16_t)3));
            else asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
        }
        __syncwarp();
    }
    if (threadIdx.x == 0) {
        while (!try_wait(smem_u32(&bar), 0)) {}
        out[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x < 32) {
        if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tm));
        else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
    }
}

int main() {
    int sms = 148;
    unsigned long long *d_out;
    CK(cudaMalloc(&d_out, sms * 8));
    std::vector<unsigned long long> h(sms);
    CK(cudaFuncSetAttribute(mma_rate<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000));
    CK(cudaFuncSetAttribute(mma_rate<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000));
    const int iters = 200;
    for (int ce : {0, 1})
    for (int N : {64, 128, 192, 256}) {
        for (int pair = 0; pair < 2; ++pair) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(sms);
            cfg.blockDim = dim3(128);
            cfg.dynamicSmemBytes = 140000;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = pair ? 2 : 1;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            for (int rep = 0; rep < 2; ++rep) {
                if (pair) CK(cudaLaunchKernelEx(&cfg, mma_rate<1>, iters, N, ce, d_out));
                else CK(cudaLaunchKernelEx(&cfg, mma_rate<0>, iters, N, ce, d_out));
            }
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(h.data(), d_out, sms * 8, cudaMemcpyDeviceToHost));
            const double cyc = (double)h[0] / (iters * 12);
            // per-SM work per instruction: 128 x N x 16 MACs either way
            printf("%s commit/4 MMAs=%d N=%3d: %.1f cycles per MMA instruction (floor 128*N/256 = %d per SM)\n",
                   pair ? "pair M=256 (cta_group::2)" : "one  M=128 (cta_group::1)", ce, N, cyc, 128 * N / 256);
        }
    }
    return 0;
}
