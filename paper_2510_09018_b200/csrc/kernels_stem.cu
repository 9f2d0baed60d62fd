// kernels_stem.cu -- the stem ("a stem convolution"): conv3x3 over the
// c_img image channels -> c0 (= ceil(r*C0)) channels, + the width's BN + ReLU, on tcgen05.
//
// K = 9*c_img (27 for RGB) is zero-padded to a multiple of 16.  The raw image's pixel stride
// (c_img*2 = 6 B) is not a TMA-addressable channel box, so the UMMA A operand (one im2col row
// per output pixel) is built in shared memory by four builder warps from a halo tile that TMA
// loads as flat image rows ([W*c_img, rows+2] box, rows outside the image zero-filled).
// Persistent, warp-specialised, one CTA per SM:
//   warp 0      TMA producer: input halo ring (4 slots)
//   warp 1      MMA issuer: NK = K/16 MMAs (M=128, N=c0) per tile into 2 TMEM accumulator stages
//   warps 4-7, 16-19  im2col builders, two tile groups: halo -> SW128 K-major A ring (4 slots)
//   warps 8-15  epilogue, two tile groups: TMEM -> fp32 BN + ReLU -> bf16 -> SW128 staging -> TMA store
// so the fetch, build, MMA and store of consecutive tiles overlap.
#include "slim_internal.h"
#include "ptx_sm100.cuh"

namespace slim {
using namespace ptx;
namespace {

constexpr int kStemThreads = 640;   // warps 0 TMA, 1 MMA, 4-7 + 16-19 im2col, 8-15 epilogue (two tile groups)
constexpr int kInSlots = 4, kASlots = 4, kAccStages = 2, kOutSlots = 2;   // slots: multiples of the 2 groups
constexpr uint32_t kInSlotBytes = 1536;   // (128/W + 2) * W * c_img * 2 <= (128 + 64) * 4 * 2

template <int CIMG>
__global__ void __launch_bounds__(kStemThreads, 1)
    stem_kernel(const __grid_constant__ CUtensorMap tmIn, const __grid_constant__ CUtensorMap tmOut, const StemArgs a) {
    constexpr int K = 9 * CIMG, NK = (K + 15) / 16;
    extern __shared__ uint8_t smem_raw[];
    // 1 KiB alignment (SW128 atoms) without leaving the shared address space
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t *pA = smem;                                   // kASlots x 128 rows x 128 B
    uint8_t *pB = pA + kASlots * 16384;                   // 64 rows x 128 B
    uint8_t *pOut = pB + 8192;                            // kOutSlots x 128 rows x 128 B
    uint8_t *pIn = pOut + kOutSlots * 16384;              // kInSlots x kInSlotBytes
    float *sBN = reinterpret_cast<float *>(pIn + kInSlots * kInSlotBytes);   // scale[64] | shift[64]
    uint64_t *bars = reinterpret_cast<uint64_t *>(sBN + 128);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * kInSlots + 2 * kASlots + 2 * kAccStages);
    const uint32_t bar0 = smem_u32(bars);
    auto in_full = [&](int i) { return bar0 + 8u * i; };
    auto in_empty = [&](int i) { return bar0 + 8u * (kInSlots + i); };
    auto a_full = [&](int i) { return bar0 + 8u * (2 * kInSlots + i); };
    auto a_empty = [&](int i) { return bar0 + 8u * (2 * kInSlots + kASlots + i); };
    auto t_full = [&](int i) { return bar0 + 8u * (2 * kInSlots + 2 * kASlots + i); };
    auto t_empty = [&](int i) { return bar0 + 8u * (2 * kInSlots + 2 * kASlots + kAccStages + i); };

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // diagnostics: td[role*64 + tile] of CTA 0 (role 0 halo issued, 1 built, 2 MMA issued, 3 stored)
    unsigned long long *td = (a.trace && blockIdx.x == 0) ? a.trace + 3584 : nullptr;
    if (td && tid == 0) td[4 * 64] = gtimer();
    const int W = a.W, rows = a.tile_rows, c0 = a.c0;
    const int acc_cols = (c0 + 31) & ~31;   // TMEM columns per accumulator stage
    const int tiles_per_img = a.H / rows;
    const uint32_t in_bytes = static_cast<uint32_t>((rows + 2) * W * CIMG * 2);

    // ---- prologue (weights and BN are not produced by the previous kernel: before the PDL wait)
    // the B tile: a straight copy of the image built at load time (rows < c0 are read)
    for (int i = tid; i < c0 * 8; i += kStemThreads)
        reinterpret_cast<uint4 *>(pB)[i] = reinterpret_cast<const uint4 *>(a.b_img)[i];
    for (int i = tid; i < c0; i += kStemThreads) {
        sBN[i] = a.scale[i];
        sBN[64 + i] = a.shift[i];
    }
    if (tid == 0) {
        for (int i = 0; i < kInSlots; ++i) {
            mbar_init(in_full(i), 1);
            mbar_init(in_empty(i), 128);
        }
        for (int i = 0; i < kASlots; ++i) {
            mbar_init(a_full(i), 128);
            mbar_init(a_empty(i), 1);
        }
        for (int i = 0; i < kAccStages; ++i) {
            mbar_init(t_full(i), 1);
            mbar_init(t_empty(i), 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_tmap(&tmIn);
        prefetch_tmap(&tmOut);
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(a.tmem_cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    fence_proxy_async();   // the generic-proxy B tile -> visible to the tensor core
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (td && tid == 0) td[4 * 64 + 1] = gtimer();
    pdl_wait();   // the output buffer may still be read by the previous kernel; the image may be its output
    pdl_launch_dependents();

    if (warp == 0) {
        // ===================== input halo producer =====================================
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int t = blockIdx.x; t < a.m_tiles; t += gridDim.x) {
                const int n = t / tiles_per_img, h0 = (t - n * tiles_per_img) * rows;
                mbar_wait(in_empty(s), ph ^ 1);
                mbar_expect_tx(in_full(s), in_bytes);
                tma_load_3d(smem_u32(pIn + s * kInSlotBytes), &tmIn, in_full(s), 0, h0 - 1, n);
                if (td) td[(t - blockIdx.x) / gridDim.x] = gtimer();
                if (++s == kInSlots) {
                    s = 0;
                    ph ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer ================================================
        const uint32_t idesc = umma_idesc_bf16(kTileM, c0);
        const uint64_t bd = umma_desc_sw128(smem_u32(pB));
        int s = 0, as = 0;
        uint32_t ph = 0, aph = 0;
        for (int t = blockIdx.x; t < a.m_tiles; t += gridDim.x) {
            mbar_wait(t_empty(as), aph ^ 1);
            mbar_wait(a_full(s), ph);
            tc_fence_after();
            if (elect_one()) {
                const uint64_t ad = umma_desc_sw128(smem_u32(pA + s * 16384));
#pragma unroll
                for (int kk = 0; kk < NK; ++kk)
                    umma_bf16(tmem + static_cast<uint32_t>(as * acc_cols), ad + 2 * kk, bd + 2 * kk, idesc, kk > 0);
                umma_commit(a_empty(s));
                umma_commit(t_full(as));
                if (td) td[2 * 64 + (t - blockIdx.x) / gridDim.x] = gtimer();
            }
            __syncwarp();
            if (++s == kASlots) {
                s = 0;
                ph ^= 1;
            }
            if (++as == kAccStages) {
                as = 0;
                aph ^= 1;
            }
        }
    } else if ((warp >= 4 && warp < 8) || warp >= 16) {
        // ===================== im2col builders: one output pixel (A row) per thread =======
        // two groups: warps 4-7 build the even tiles, 16-19 the odd ones (input / A slots
        // ti mod 4 are then always the same group's, so the parity waits stay in order)
        const int bg = warp >= 16 ? 1 : 0;
        const int row = tid - (bg ? 512 : 128), sw = row & 7;
        const int r_pix = row / W, c_pix = row - r_pix * W;
        for (int t = blockIdx.x + bg * gridDim.x; t < a.m_tiles; t += 2 * gridDim.x) {
            const int ti = (t - blockIdx.x) / gridDim.x;
            const int s = ti % kInSlots, as = ti % kASlots;
            const uint32_t ph = (ti / kInSlots) & 1, aph = (ti / kASlots) & 1;
            mbar_wait(in_full(s), ph);
            const uint16_t *hb = reinterpret_cast<const uint16_t *>(pIn + s * kInSlotBytes);
            uint32_t packed[NK * 8];
#pragma unroll
            for (int j = 0; j < NK * 8; ++j) packed[j] = 0;
#pragma unroll
            for (int kh = 0; kh < 3; ++kh)
#pragma unroll
                for (int kw = 0; kw < 3; ++kw) {
                    const int col = c_pix + kw - 1;
                    const bool ok = col >= 0 && col < W;
                    const uint16_t *px = hb + ((r_pix + kh) * W + col) * CIMG;
#pragma unroll
                    for (int ci = 0; ci < CIMG; ++ci) {
                        const int k = (kh * 3 + kw) * CIMG + ci;
                        const uint32_t b = ok ? static_cast<uint32_t>(px[ci]) : 0u;
                        packed[k >> 1] |= (k & 1) ? (b << 16) : b;
                    }
                }
            mbar_arrive(in_empty(s));   // halo slot consumed
            mbar_wait(a_empty(as), aph ^ 1);
            uint8_t *dst = pA + as * 16384 + row * 128;
#pragma unroll
            for (int j = 0; j < NK * 2; ++j)   // 16-B piece j holds K = 8j .. 8j+7
                *reinterpret_cast<uint4 *>(dst + ((j ^ sw) << 4)) =
                    make_uint4(packed[4 * j], packed[4 * j + 1], packed[4 * j + 2], packed[4 * j + 3]);
            fence_proxy_async();        // generic smem writes -> visible to the tensor core
            mbar_arrive(a_full(as));
            if (td && row == 0) td[64 + ti] = gtimer();
        }
    } else if (warp >= 8 && warp < 16) {
        // ===================== epilogue: warps 8-11 take the even tiles, 12-15 the odd ones ====
        const int grp = (warp - 8) >> 2;
        const int q = warp & 3, row = q * 32 + lane, sw = row & 7;
        const bool leader = (warp == 8 + 4 * grp && lane == 0);
        const uint32_t lane_addr = tmem + (static_cast<uint32_t>(q * 32) << 16);
        uint8_t *pOutG = pOut + grp * 16384;   // staging slot of this group
        for (int t = blockIdx.x + grp * gridDim.x; t < a.m_tiles; t += 2 * gridDim.x) {
            const int n = t / tiles_per_img, h0 = (t - n * tiles_per_img) * rows;
            const int ti = (t - blockIdx.x) / gridDim.x;
            const int as = ti & 1;                          // accumulator stage = tile parity = group
            const uint32_t aph = (ti >> 1) & 1;
            mbar_wait(t_full(as), aph);
            tc_fence_after();
            if (leader) bulk_wait_read0();   // this group's previous store has left the staging slot
            named_bar_sync(1 + grp, 128);
            uint8_t *rowp = pOutG + row * 128;
            for (int g = 0; g < c0 / 16; ++g) {
                uint32_t v[16];
                tmem_ld16(lane_addr + static_cast<uint32_t>(as * acc_cols + g * 16), v);
                tmem_wait_ld();
                reg_fence16(v);
                float f[16];
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    f[i] = fmaxf(fmaf(__uint_as_float(v[i]), sBN[g * 16 + i], sBN[64 + g * 16 + i]), a.relu_lo);
                const int q16 = g * 2;
                *reinterpret_cast<uint4 *>(rowp + ((q16 ^ sw) << 4)) =
                    make_uint4(pack_bf16(f[0], f[1]), pack_bf16(f[2], f[3]), pack_bf16(f[4], f[5]), pack_bf16(f[6], f[7]));
                *reinterpret_cast<uint4 *>(rowp + (((q16 + 1) ^ sw) << 4)) = make_uint4(
                    pack_bf16(f[8], f[9]), pack_bf16(f[10], f[11]), pack_bf16(f[12], f[13]), pack_bf16(f[14], f[15]));
            }
            tc_fence_before();
            mbar_arrive(t_empty(as));
            fence_proxy_async();
            named_bar_sync(1 + grp, 128);
            if (leader) {
                tma_store_4d(&tmOut, smem_u32(pOutG), 0, 0, h0, n);
                bulk_commit();
                if (td) td[3 * 64 + ti] = gtimer();
            }
        }
        if (leader) bulk_wait0();
    }
    tc_fence_before();
    __syncthreads();
    if (td && tid == 0) td[4 * 64 + 2] = gtimer();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols) : "memory");
    }
}

size_t stem_smem_bytes() {
    return 1024 + kASlots * 16384 + 8192 + kOutSlots * 16384 + kInSlots * kInSlotBytes + 128 * 4 +
           8 * (2 * kInSlots + 2 * kASlots + 2 * kAccStages) + 16;
}

}  // namespace

cudaError_t launch_stem_umma(const StemArgs &a, const CUtensorMap &tmIn, const CUtensorMap &tmOut, int grid,
                             cudaStream_t stream, bool pdl) {
    using Fn = void (*)(CUtensorMap, CUtensorMap, StemArgs);
    Fn fn = a.cimg == 1 ? stem_kernel<1> : a.cimg == 2 ? stem_kernel<2> : a.cimg == 3 ? stem_kernel<3> : stem_kernel<4>;
    static bool attr_set = false;
    if (!attr_set) {
        const Fn all[4] = {stem_kernel<1>, stem_kernel<2>, stem_kernel<3>, stem_kernel<4>};
        for (Fn f : all) {
            cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(stem_smem_bytes()));
            if (e != cudaSuccess) return e;
        }
        attr_set = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kStemThreads);
    cfg.dynamicSmemBytes = stem_smem_bytes();
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, fn, tmIn, tmOut, a);
}

}  // namespace slim
