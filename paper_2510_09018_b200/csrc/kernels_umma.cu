// kernels_umma.cu -- width-sliced implicit-GEMM convolution on sm_100a tensor cores.
//
// The hot path of the paper's method: the batched forward of a segment of the
// universally slimmable SlimResNet at width r.  A conv3x3 / conv1x1
// over the first c_in = c(r_prev) input and c_out = c(r) output channels of the
// FULL-width shared weights, followed by the fused epilogue
//     relu( s[c]*acc + t[c]  [+ residual]  [+ s_sc[c]*acc_sc + t_sc[c]] )
// where (s, t) is the switchable BN of this width folded on the host (north_star).
//
// GEMM mapping:
//   M = B*Ho*Wo output pixels in NHWC order, one CTA tile = 128 consecutive pixels
//       (tile_imgs images x tile_rows rows x Wo columns),
//   N = c_out (n_tile <= 256 per tile), K = k*k*c_in, iterated as K-blocks of
//       (filter tap, 64-channel chunk).
//   A tile (128 x 64 bf16) = a 4-D TMA box of the NHWC input at the tap's shifted
//       origin; zero padding and the stride-2 subsampling are done by the TMA unit
//       (negative / out-of-range coordinates fill 0, elementStrides = stride).
//   B tile (n_tile x 64 bf16) = a 3-D TMA box of the KRSC weights whose tensor-map
//       bounds are the ACTIVE prefix (c_in, c_out): channels beyond the prefix
//       are never read -- "tile predication, not copying weights" (north_star).
//   D = FP32 accumulator in TMEM (lane = pixel row, column = channel), double
//       buffered across tiles so the epilogue of tile i overlaps the MMAs of i+1.
// Warp roles (192 threads, persistent over tiles): warp 0 = TMA producer,
// warp 1 = TMEM allocator + single-thread tcgen05.mma issuer, warps 2..5 =
// epilogue (tcgen05.ld -> BN/residual/ReLU in fp32 -> bf16 -> swizzled smem ->
// TMA store; the residual tile arrives by TMA into the same staging buffer).
#include "slim_internal.h"

#include <cuda_bf16.h>

#include <map>
#include <mutex>

namespace slim {
namespace {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier ---------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// ---- TMA ----------------------------------------------------------------------
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap *tm, uint32_t bar, int c0, int c1,
                                            int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap *tm, uint32_t bar, int c0, int c1,
                                            int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap *tm, uint32_t src, int c0, int c1, int c2, int c3) {
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(tm)),
                 "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *tm) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tm)) : "memory");
}

// ---- tcgen05 ------------------------------------------------------------------
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Shared-memory matrix descriptor, K-major, 128-byte swizzle (SM100 "version 1"):
// start>>4 [0,14), LBO>>4 [16,30) (=1, unused for swizzled K-major), SBO>>4 [32,46)
// (= 1024 B between 8-row core-matrix groups), version [46,48) = 1, layout [61,64) = 2.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>(1) << 16;
    d |= static_cast<uint64_t>(1024 >> 4) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(2) << 61;
    return d;
}
// Instruction descriptor kind::f16: D=f32 [4,6)=1, A=bf16 [7,10)=1, B=bf16 [10,13)=1,
// both K-major, N>>3 at [17,23), M>>4 at [24,29).
__device__ __forceinline__ uint32_t umma_idesc_bf16(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
           (static_cast<uint32_t>(M >> 4) << 24);
}
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);   // RNE, one rounding per stored value
    return *reinterpret_cast<uint32_t *>(&h);
}
__device__ __forceinline__ float bf16_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t u) { return __uint_as_float(u & 0xFFFF0000u); }

struct TileCoord {
    int n0, h0, co0;
};
__device__ __forceinline__ TileCoord tile_coord(const ConvArgs &a, int t) {
    const int mt = t % a.m_tiles, nt = t / a.m_tiles;
    TileCoord c;
    if (a.tile_imgs == 1) {
        c.n0 = mt / a.tiles_per_img;
        c.h0 = (mt % a.tiles_per_img) * a.tile_rows;
    } else {
        c.n0 = mt * a.tile_imgs;
        c.h0 = 0;
    }
    c.co0 = nt * a.n_tile;
    return c;
}

__global__ void __launch_bounds__(kConvThreads, 1)
    conv_umma_kernel(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmB0,
                     const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmB1,
                     const __grid_constant__ CUtensorMap tmRes, const __grid_constant__ CUtensorMap tmOut,
                     const ConvArgs a) {
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment: SW128 TMA boxes and UMMA descriptors (base_offset = 0)
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = a.n_stages;
    const uint32_t sA = smem_u32(smem);
    const uint32_t sB = sA + S * kTileABytes;
    const uint32_t sOut = sB + S * a.stage_b_bytes;
    uint8_t *pOut = smem + (sOut - sA);
    uint64_t *bars = reinterpret_cast<uint64_t *>(pOut + a.n_out_chunks * 16384);
    const uint32_t bar0 = smem_u32(bars);
    // barrier map: full[0,S) empty[S,2S) tmem_full[2S,2S+2) tmem_empty[2S+2,2S+4) res[2S+4]
    auto full_bar = [&](int i) { return bar0 + 8u * i; };
    auto empty_bar = [&](int i) { return bar0 + 8u * (S + i); };
    auto tfull_bar = [&](int i) { return bar0 + 8u * (2 * S + i); };
    auto tempty_bar = [&](int i) { return bar0 + 8u * (2 * S + 2 + i); };
    const uint32_t res_bar = bar0 + 8u * (2 * S + 4);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * S + 5);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int total = a.m_tiles * a.n_tiles;

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(full_bar(i), 1);
            mbar_init(empty_bar(i), 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(tfull_bar(i), 1);
            mbar_init(tempty_bar(i), 128);
        }
        mbar_init(res_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_tmap(&tmA0);
        prefetch_tmap(&tmB0);
        if (a.n_parts > 1) {
            prefetch_tmap(&tmA1);
            prefetch_tmap(&tmB1);
        }
        prefetch_tmap(&tmOut);
        if (a.epi == EPI_BN_ADD_RELU) prefetch_tmap(&tmRes);
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(a.tmem_cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ===================== TMA producer (one thread) =====================
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            const uint32_t tx = kTileABytes + a.stage_b_bytes;
            for (int t = blockIdx.x; t < total; t += gridDim.x) {
                const TileCoord tc = tile_coord(a, t);
                for (int p = 0; p < a.n_parts; ++p) {
                    const GemmPart &gp = a.part[p];
                    const CUtensorMap *tA = p ? &tmA1 : &tmA0;
                    const CUtensorMap *tB = p ? &tmB1 : &tmB0;
                    for (int kb = 0; kb < gp.n_kblocks; ++kb) {
                        const int tap = kb / gp.n_chunks, ch = kb - tap * gp.n_chunks;
                        const int kh = tap / gp.ksize, kw = tap - kh * gp.ksize;
                        mbar_wait(empty_bar(stage), phase ^ 1);
                        mbar_expect_tx(full_bar(stage), tx);
                        tma_load_4d(sA + stage * kTileABytes, tA, full_bar(stage), ch * kChunk, kw - gp.pad,
                                    tc.h0 * gp.stride + kh - gp.pad, tc.n0);
                        tma_load_3d(sB + stage * a.stage_b_bytes, tB, full_bar(stage), ch * kChunk, tap, tc.co0);
                        if (++stage == S) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (one thread) =======================
        if (lane == 0) {
            const uint32_t idesc = umma_idesc_bf16(kTileM, a.n_tile);
            int stage = 0, as = 0;
            uint32_t phase = 0, aphase = 0;
            for (int t = blockIdx.x; t < total; t += gridDim.x) {
                mbar_wait(tempty_bar(as), aphase ^ 1);
                tc_fence_after();
                for (int p = 0; p < a.n_parts; ++p) {
                    const GemmPart &gp = a.part[p];
                    const uint32_t d = tmem_base + static_cast<uint32_t>((as * a.n_parts + p) * a.acc_stride);
                    for (int kb = 0; kb < gp.n_kblocks; ++kb) {
                        const int ch = kb % gp.n_chunks;
                        int nk = (gp.c_in - ch * kChunk + 15) >> 4;
                        nk = nk > 4 ? 4 : nk;
                        mbar_wait(full_bar(stage), phase);
                        tc_fence_after();
                        const uint64_t ad = umma_desc_sw128(sA + stage * kTileABytes);
                        const uint64_t bd = umma_desc_sw128(sB + stage * a.stage_b_bytes);
                        for (int kk = 0; kk < nk; ++kk)   // K=16 per MMA = 32 bytes inside the 128-B atom
                            umma_bf16(d, ad + 2 * kk, bd + 2 * kk, idesc, (kb | kk) != 0);
                        umma_commit(empty_bar(stage));   // frees the smem slot when these MMAs finish
                        if (++stage == S) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
                umma_commit(tfull_bar(as));   // accumulator ready for the epilogue
                if (++as == a.acc_stages) {
                    as = 0;
                    aphase ^= 1;
                }
            }
        }
    } else {
        // ===================== epilogue (warps 2..5) =========================
        const int q = warp & 3;              // TMEM lane quarter this warp may access
        const int row = q * 32 + lane;       // pixel row inside the 128-pixel tile
        const bool leader = (warp == 2 && lane == 0);
        const uint32_t lane_addr = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
        const int sw = row & 7;
        int as = 0;
        uint32_t aphase = 0, rphase = 0;
        for (int t = blockIdx.x; t < total; t += gridDim.x) {
            const TileCoord tc = tile_coord(a, t);
            mbar_wait(tfull_bar(as), aphase);
            tc_fence_after();
            if (leader) bulk_wait_read0();   // previous tile's stores have left the staging buffer
            if (a.epi == EPI_BN_ADD_RELU) {
                if (leader) {
                    mbar_expect_tx(res_bar, a.n_out_chunks * 16384u);
                    for (uint32_t j = 0; j < a.n_out_chunks; ++j)
                        tma_load_4d(sOut + j * 16384u, &tmRes, res_bar, tc.co0 + j * kChunk, 0, tc.h0, tc.n0);
                }
                mbar_wait(res_bar, rphase);
                rphase ^= 1;
            } else {
                named_bar_sync(1, 128);
            }
            const uint32_t col0 = static_cast<uint32_t>(as * a.n_parts * a.acc_stride);
            for (int g = 0; g < a.n_tile / 16; ++g) {
                uint32_t v[16], u[16];
                tmem_ld16(lane_addr + col0 + g * 16, v);
                if (a.epi == EPI_BN_PROJ_RELU) tmem_ld16(lane_addr + col0 + a.acc_stride + g * 16, u);
                tmem_wait_ld();
                const int cl = g * 16;             // channel inside the tile
                const int cg = tc.co0 + cl;        // global output channel
                float f[16];
                const float4 *s4 = reinterpret_cast<const float4 *>(a.scale0 + cg);
                const float4 *t4 = reinterpret_cast<const float4 *>(a.shift0 + cg);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float4 s = __ldg(s4 + i), b = __ldg(t4 + i);
                    f[4 * i + 0] = fmaf(__uint_as_float(v[4 * i + 0]), s.x, b.x);
                    f[4 * i + 1] = fmaf(__uint_as_float(v[4 * i + 1]), s.y, b.y);
                    f[4 * i + 2] = fmaf(__uint_as_float(v[4 * i + 2]), s.z, b.z);
                    f[4 * i + 3] = fmaf(__uint_as_float(v[4 * i + 3]), s.w, b.w);
                }
                if (a.epi == EPI_BN_PROJ_RELU) {
                    const float4 *s14 = reinterpret_cast<const float4 *>(a.scale1 + cg);
                    const float4 *t14 = reinterpret_cast<const float4 *>(a.shift1 + cg);
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const float4 s = __ldg(s14 + i), b = __ldg(t14 + i);
                        f[4 * i + 0] += fmaf(__uint_as_float(u[4 * i + 0]), s.x, b.x);
                        f[4 * i + 1] += fmaf(__uint_as_float(u[4 * i + 1]), s.y, b.y);
                        f[4 * i + 2] += fmaf(__uint_as_float(u[4 * i + 2]), s.z, b.z);
                        f[4 * i + 3] += fmaf(__uint_as_float(u[4 * i + 3]), s.w, b.w);
                    }
                }
                // staging: chunk cl/64, row `row`, 16-B pieces (cl%64)/8 and +1, SW128 swizzled
                uint8_t *rowp = pOut + (cl >> 6) * 16384 + row * 128;
                const int q16 = (cl & 63) >> 3;
                uint4 *p0 = reinterpret_cast<uint4 *>(rowp + (((q16) ^ sw) << 4));
                uint4 *p1 = reinterpret_cast<uint4 *>(rowp + (((q16 + 1) ^ sw) << 4));
                if (a.epi == EPI_BN_ADD_RELU) {
                    const uint4 r0 = *p0, r1 = *p1;
                    const uint32_t rr[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        f[2 * i] += bf16_lo(rr[i]);
                        f[2 * i + 1] += bf16_hi(rr[i]);
                    }
                }
                uint32_t o[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) o[i] = pack_bf16(fmaxf(f[2 * i], 0.f), fmaxf(f[2 * i + 1], 0.f));
                *p0 = make_uint4(o[0], o[1], o[2], o[3]);
                *p1 = make_uint4(o[4], o[5], o[6], o[7]);
            }
            tc_fence_before();
            mbar_arrive(tempty_bar(as));     // TMEM accumulator may be overwritten
            fence_proxy_async();             // generic smem writes -> visible to the TMA (async proxy)
            named_bar_sync(1, 128);
            if (leader) {
                for (uint32_t j = 0; j < a.n_out_chunks; ++j)
                    tma_store_4d(&tmOut, sOut + j * 16384u, tc.co0 + j * kChunk, 0, tc.h0, tc.n0);
                bulk_commit();
            }
            if (++as == a.acc_stages) {
                as = 0;
                aphase ^= 1;
            }
        }
        if (leader) bulk_wait0();
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(a.tmem_cols)
                     : "memory");
    }
}

}  // namespace

size_t conv_umma_smem_bytes(const ConvArgs &a) {
    return 1024 /*alignment slack*/ + static_cast<size_t>(a.n_stages) * (kTileABytes + a.stage_b_bytes) +
           static_cast<size_t>(a.n_out_chunks) * 16384 + 8 * (2 * kMaxStages + 5) + 16;
}

int conv_umma_max_ctas_per_sm(size_t smem_bytes) {
    // cached per shared-memory size: the occupancy query costs microseconds of host time
    static std::mutex mu;
    static std::map<size_t, int> cache;
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(smem_bytes);
    if (it != cache.end()) return it->second;
    int n = 0;
    cudaFuncSetAttribute(conv_umma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, conv_umma_kernel, kConvThreads, smem_bytes) != cudaSuccess) {
        cudaGetLastError();
        n = 1;
    }
    n = n < 1 ? 1 : n;
    cache[smem_bytes] = n;
    return n;
}

cudaError_t launch_conv_umma(const ConvArgs &a, const CUtensorMap &tmA0, const CUtensorMap &tmB0,
                             const CUtensorMap &tmA1, const CUtensorMap &tmB1, const CUtensorMap &tmRes,
                             const CUtensorMap &tmOut, int grid, cudaStream_t stream) {
    const size_t smem = conv_umma_smem_bytes(a);
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(conv_umma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    conv_umma_kernel<<<grid, kConvThreads, smem, stream>>>(tmA0, tmB0, tmA1, tmB1, tmRes, tmOut, a);
    return cudaGetLastError();
}

}  // namespace slim
