// Microbenchmarks of the two primitives the conv kernel is built on (diagnostic tool,
// not part of libslim): (1) back-to-back tcgen05.mma issue rate from smem operands,
// (2) TMA 4-D box load throughput per SM for the conv's A-tile box shape.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench ubench.cu -lcuda
#include <cuda.h>
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

// (1) MMA issue rate.  variant 0: lane 0 alone runs the loop (divergent);
// variant 1: the whole warp runs a warp-uniform loop and one elected lane issues
// (CUTLASS/DeepGEMM style), inner 4 K-steps unrolled, 3 accumulators x 3 A offsets.
__device__ __forceinline__ uint32_t elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n .reg .b32 r;\n .reg .pred p;\n elect.sync r|p, 0xffffffff;\n selp.u32 %0, 1, 0, p;\n}" : "=r"(pred));
    return pred;
}
__device__ __forceinline__ void mma_issue(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__global__ void mma_rate(int n_iter, int N, int variant, unsigned long long *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *s = (uint8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tslot;
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t ad = desc_sw128(smem_u32(s)), bd = desc_sw128(smem_u32(s + 32768));
    unsigned long long t0 = clock64();
    if (variant == 0) {
        if (threadIdx.x == 0) {
            for (int it = 0; it < n_iter; ++it)
                for (int kh = 0; kh < 3; ++kh)
                    for (int kw = 0; kw < 3; ++kw)
                        for (int kk = 0; kk < 4; ++kk)
                            mma_issue(tm + kw * N, ad + kh * 256 + 2 * kk, bd + kw * 64 + 2 * kk, idesc, (it | kh | kk) != 0);
        }
    } else if (variant == 2 && threadIdx.x < 32) {
        // uniform loop, ONE elect around the whole batch of MMAs (CUTLASS style)
        for (int it = 0; it < n_iter; ++it) {
            if (elect_one()) {
#pragma unroll
                for (int kh = 0; kh < 3; ++kh)
#pragma unroll
                    for (int kw = 0; kw < 3; ++kw)
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            mma_issue(tm + kw * N, ad + kh * 256 + 2 * kk, bd + kw * 64 + 2 * kk, idesc, (it | kh | kk) != 0);
            }
            __syncwarp();
        }
    } else if (threadIdx.x < 32) {
        for (int it = 0; it < n_iter; ++it) {
#pragma unroll
            for (int kh = 0; kh < 3; ++kh)
#pragma unroll
                for (int kw = 0; kw < 3; ++kw)
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        if (elect_one()) mma_issue(tm + kw * N, ad + kh * 256 + 2 * kk, bd + kw * 64 + 2 * kk, idesc, (it | kh | kk) != 0);
            __syncwarp();
        }
    }
    if (threadIdx.x == 0) {
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
        while (!try_wait(smem_u32(&bar), 0)) {}
        out[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

// (2) TMA throughput: `issuers` threads each stream n_loads boxes through their own ring of
// `stages` slots (slot released as soon as its bytes land; no consumer work).
__global__ void tma_rate(const __grid_constant__ CUtensorMap tm, int rank, int n_loads, int stages, int box_bytes,
                         int ntiles, int issuers, int uniform, unsigned long long *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *s = (uint8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bars[4][16];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int j = 0; j < issuers; ++j)
            for (int i = 0; i < stages; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[j][i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    unsigned long long t0 = clock64();
    if (w < issuers && (uniform || lane == 0)) {
        uint8_t *base = s + w * stages * box_bytes;
        for (int i = 0; i < n_loads; ++i) {
            int st = i % stages;
            if (i >= stages) while (!try_wait(smem_u32(&bars[w][st]), ((i / stages) - 1) & 1)) {}
            uint32_t b = smem_u32(&bars[w][st]);
            const bool me = uniform ? elect_one() : true;
            if (me) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(box_bytes));
            int tile = (blockIdx.x * issuers + w + i * gridDim.x * issuers) % ntiles;
            uint32_t dst = smem_u32(base + st * box_bytes);
            if (!me) { __syncwarp(); continue; }
            if (rank == 4) {
                int n = tile / 8, h0 = (tile % 8) * 4;
                int kw = i % 3 - 1, kh = (i / 3) % 3 - 1;
                asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                             ::"r"(dst), "l"((uint64_t)&tm), "r"(b), "r"(0), "r"(kw), "r"(h0 + kh), "r"(n) : "memory");
            } else {
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                             ::"r"(dst), "l"((uint64_t)&tm), "r"(b), "r"(0), "r"(tile * 128) : "memory");
            }
            if (uniform) __syncwarp();
        }
        for (int i = n_loads - stages; i < n_loads; ++i) {
            int st = i % stages;
            while (!try_wait(smem_u32(&bars[w][st]), (i / stages) & 1)) {}
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*EncFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                          const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    unsigned long long *d_out; CK(cudaMalloc(&d_out, 4096 * 8));
    std::vector<unsigned long long> h(4096);
    CK(cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000));
    for (int variant = 0; variant < 3; ++variant)
        for (int N : {16, 64, 128}) {
            for (int rep = 0; rep < 2; ++rep) mma_rate<<<sms, 128, 70000>>>(100, N, variant, d_out);
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(h.data(), d_out, sms * 8, cudaMemcpyDeviceToHost));
            double cyc = (double)h[0] / (100 * 36);
            printf("MMA variant %d M=128 N=%3d K=16 (3 acc x 3 A offsets): %.1f cycles/instr (floor %d)\n", variant, N, cyc, 128 * N / 256);
        }
    void *fn; cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    EncFn enc = (EncFn)fn;
    CK(cudaFuncSetAttribute(tma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 220000));
    const int B = 128, C = 64;
    void *act; CK(cudaMalloc(&act, (size_t)B * 32 * 32 * C * 2));
    CK(cudaMemset(act, 0, (size_t)B * 32 * 32 * C * 2));
    struct Cfg { const char *name; int rank; int inner; int rows; CUtensorMapSwizzle sw; };
    Cfg cfgs[] = {{"4D [64,32,4,1] SW128", 4, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B},
                  {"2D [64,128] SW128", 2, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B},
                  {"2D [64,256] SW128", 2, 64, 256, CU_TENSOR_MAP_SWIZZLE_128B},

                  };
    for (auto &c : cfgs) {
        CUtensorMap tm;
        CUresult r;
        if (c.rank == 4) {
            cuuint64_t dims[4] = {(cuuint64_t)C, 32, 32, (cuuint64_t)B};
            cuuint64_t str[3] = {(cuuint64_t)C * 2, (cuuint64_t)32 * C * 2, (cuuint64_t)32 * 32 * C * 2};
            cuuint32_t box[4] = {64, 32, 4, 1}, es[4] = {1, 1, 1, 1};
            r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, act, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, c.sw,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {
            cuuint64_t total = (cuuint64_t)B * 32 * 32 * C;
            cuuint64_t dims[2] = {(cuuint64_t)c.inner, total / c.inner};
            cuuint64_t str[1] = {(cuuint64_t)c.inner * 2};
            cuuint32_t box[2] = {(cuuint32_t)c.inner, (cuuint32_t)c.rows}, es[2] = {1, 1};
            r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, act, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, c.sw,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        if (r != CUDA_SUCCESS) { printf("%s: encode failed %d\n", c.name, r); continue; }
        int bb = c.inner * c.rows * 2;
        int ntiles = (int)((size_t)B * 32 * 32 * C * 2 / bb) - 2;
        for (int uniform : {0, 1})
        for (int issuers : {1, 2}) {
            int stages = 6;
            if (issuers * stages * bb + 1024 > 220000) stages = (220000 - 1024) / (issuers * bb);
            for (int rep = 0; rep < 2; ++rep)
                tma_rate<<<sms, 128, issuers * stages * bb + 1024>>>(tm, c.rank, 200, stages, bb, ntiles, issuers, uniform, d_out);
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(h.data(), d_out, sms * 8, cudaMemcpyDeviceToHost));
            double cyc = 0; for (int i = 0; i < sms; ++i) cyc += h[i]; cyc /= sms;
            double bpc = 200.0 * issuers * bb / cyc;
            printf("TMA %-22s uniform=%d issuers=%d stages=%2d: %6.1f B/cycle/SM (%.2f TB/s chip)\n", c.name, uniform, issuers, stages, bpc,
                   bpc * sms * clk * 1e3 / 1e12);
        }
    }
    return 0;
}
