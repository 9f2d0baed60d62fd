// kernels_splitk.cu -- split-K width-sliced conv for the small-M late segments (tcgen05 + DSMEM).
//
// Same operation as conv_umma_kernel (kernels_umma.cu):
//     out = relu( s*conv(x) + t  [+ residual]  [+ s_sc*proj(x_sc) + t_sc] )   [-> fused avg pool]
// over the active channel prefixes of the shared full-width weights (north_star).
//
// Why a second kernel: in segments 2-3 M = B*Ho*Wo is small (2048 rows at B=128 in seg 3) and K
// is large (9*512), so covering the SMs with 128 x 64 tiles re-reads every A tile n_tiles times
// and every B tile m_tiles times -- the L2->SM traffic (not the tensor core) bounds the layer.
// Here one output tile is 128 x n_tile with n_tile up to 256 (one UMMA N) and the K range is
// split over the ks CTAs of a thread-block cluster: 2-4x fewer bytes per output than the
// narrow tiles at the same CTA count.  The ks fp32 partial tiles are reduced through
// distributed shared memory: CTA r owns output channels [r*w_o, (r+1)*w_o) of the tile; every
// CTA pushes its TMEM partial of the other owners' slices into their shared memory (reusing the
// drained pipeline stages), and each owner sums the ks partials in rank order 0..ks-1 -- a
// fixed order, so the result does not depend on timing or batch size (ks is chosen from the
// layer shape and the context's max_batch only).
//
// Roles (384 threads, one tile per CTA): warps 0, 2, 3 = TMA producers (k-block round robin),
// warp 1 = TMEM allocator + MMA issuer, warps 4..11 = epilogue / reduction (two per TMEM lane
// quarter, alternating 16-column groups).
#include "slim_internal.h"
#include "ptx_sm100.cuh"

namespace slim {
using namespace ptx;
namespace {

constexpr int kSplitThreads = 384;

__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared::cluster.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}

__global__ void __launch_bounds__(kSplitThreads, 1)
    conv_splitk_kernel(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmB0,
                       const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmB1,
                       const __grid_constant__ CUtensorMap tmRes, const __grid_constant__ CUtensorMap tmOut,
                       const SplitArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int S = a.n_stages, KS = a.ks, NT = a.n_tile, WO = a.w_o;
    const uint32_t stage_bytes = a.stage_bytes;
    const uint32_t oc_bytes = 128u * a.rbo;
    const uint32_t slice_bytes = a.n_out_chunks * oc_bytes;   // owner slice: 128 pixels x w_o bf16
    uint8_t *pStage = smem;
    uint8_t *pOut = pStage + S * stage_bytes;
    uint8_t *pRes = pOut + slice_bytes;
    const bool has_res = a.epi == EPI_BN_ADD_RELU;
    float *sBN = reinterpret_cast<float *>(pRes + (has_res ? slice_bytes : 0));   // s0|t0|s1|t1 of the owner slice
    uint64_t *bars = reinterpret_cast<uint64_t *>(sBN + 4 * WO);
    const uint32_t bar0 = smem_u32(bars);
    auto full_bar = [&](int i) { return bar0 + 8u * i; };
    auto empty_bar = [&](int i) { return bar0 + 8u * (S + i); };
    const uint32_t tfull = bar0 + 8u * (2 * S), rfull = bar0 + 8u * (2 * S + 1);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * S + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rank = static_cast<int>(cluster_ctarank());
    const int tile = static_cast<int>(blockIdx.x) / KS;
    const int mt = tile % a.m_tiles, ntile = tile / a.m_tiles;
    int n0, h0;
    if (a.tile_imgs == 1) {
        n0 = mt / a.tiles_per_img;
        h0 = (mt % a.tiles_per_img) * a.tile_rows;
    } else {
        n0 = mt * a.tile_imgs;
        h0 = 0;
    }
    const int co_tile = ntile * NT;            // first output channel of the tile
    const int co_own = co_tile + rank * WO;    // first output channel this CTA finishes

    // k-blocks of the tile: part 0 (taps x 64-channel chunks) then part 1 (projection chunks);
    // this CTA takes the contiguous range [g0, g1)
    const int G0 = a.part[0].n_kblocks, G = G0 + (a.n_parts > 1 ? a.part[1].n_kblocks : 0);
    const int g0 = rank * G / KS, g1 = (rank + 1) * G / KS;

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(full_bar(i), 1);
            mbar_init(empty_bar(i), 1);
        }
        mbar_init(tfull, 1);
        mbar_init(rfull, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_tmap(&tmA0);
        prefetch_tmap(&tmB0);
        if (a.n_parts > 1) {
            prefetch_tmap(&tmA1);
            prefetch_tmap(&tmB1);
        }
        if (!a.pool_out) prefetch_tmap(&tmOut);
        if (has_res) prefetch_tmap(&tmRes);
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(a.tmem_cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    for (int i = threadIdx.x; i < WO; i += blockDim.x) {
        sBN[i] = a.scale0[co_own + i];
        sBN[WO + i] = a.shift0[co_own + i];
        if (a.n_parts > 1) {
            sBN[2 * WO + i] = a.scale1[co_own + i];
            sBN[3 * WO + i] = a.shift1[co_own + i];
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_wait();
    pdl_launch_dependents();

    if (warp == 0 || warp == 2 || warp == 3) {
        // ===================== TMA producers ===============================================
        const int pi = warp == 0 ? 0 : warp - 1;
        if (lane == 0 && pi < a.n_prod) {
            if (pi == 0 && has_res) {   // the owner slice of the residual, once
                mbar_expect_tx(rfull, slice_bytes);
                for (uint32_t j = 0; j < a.n_out_chunks; ++j)
                    tma_load_4d(smem_u32(pRes + j * oc_bytes), &tmRes, rfull, co_own + j * a.co_chunk, 0, h0, n0);
            }
            const uint32_t b_bytes = static_cast<uint32_t>(NT) * 128u;
            for (int g = g0; g < g1; ++g) {
                const int l = g - g0;
                if (l % a.n_prod != pi) continue;
                const int stage = l % S;
                const uint32_t phase = (l / S) & 1;
                mbar_wait(empty_bar(stage), phase ^ 1);
                mbar_expect_tx(full_bar(stage), 16384u + b_bytes);
                const int p = g < G0 ? 0 : 1;
                const int nch = p ? a.part[1].n_chunks : a.part[0].n_chunks;
                const int ksz = p ? a.part[1].ksize : a.part[0].ksize;
                const int gpad = p ? a.part[1].pad : a.part[0].pad;
                const int gstr = p ? a.part[1].stride : a.part[0].stride;
                const int kb = p ? g - G0 : g;
                const int tap = kb / nch, ch = kb - tap * nch;
                const int kh = tap / ksz, kw = tap - kh * ksz;
                const uint32_t sA = smem_u32(pStage + stage * stage_bytes);
                tma_load_4d(sA, p ? &tmA1 : &tmA0, full_bar(stage), ch * kChunk, kw - gpad, h0 * gstr + kh - gpad, n0);
                tma_load_3d(sA + 16384u, p ? &tmB1 : &tmB0, full_bar(stage), ch * kChunk, tap, co_tile);
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =================================================
        const uint32_t idesc = umma_idesc_bf16(kTileM, NT);
        const uint64_t desc0 = umma_desc_kmajor(smem_u32(pStage), 128);
        const uint32_t stage16 = stage_bytes >> 4;
        for (int g = g0; g < g1; ++g) {
            const int l = g - g0;
            const int stage = l % S;
            const uint32_t phase = (l / S) & 1;
            const int p = g < G0 ? 0 : 1;
            const int nch = p ? a.part[1].n_chunks : a.part[0].n_chunks;
            const int cin = p ? a.part[1].c_in : a.part[0].c_in;
            const int kb = p ? g - G0 : g;
            const int ch = kb % nch;
            const int nk = min(4, (cin - ch * kChunk + 15) >> 4);
            // first k-block of this part in this CTA's range starts the accumulator
            const bool first = (g == g0) || (p == 1 && g == G0);
            mbar_wait(full_bar(stage), phase);
            tc_fence_after();
            if (elect_one()) {
                const uint64_t ad = desc0 + stage * stage16;
                const uint64_t bd = ad + (16384u >> 4);
                const uint32_t d = tmem_base + static_cast<uint32_t>(p * NT);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    if (kk < nk) umma_bf16(d, ad + 2 * kk, bd + 2 * kk, idesc, !(first && kk == 0));
                umma_commit(empty_bar(stage));
            }
            __syncwarp();
        }
        if (elect_one()) umma_commit(tfull);
        __syncwarp();
    }

    // ===================== split-K reduction over the cluster (DSMEM) =====================
    // The epilogue warps wait for this CTA's MMAs; after barrier 1 every CTA's pipeline stages
    // are drained and serve as its receive buffer recv[slot][part][g16][piece][row] (fp32 x 4).
    const bool epi = warp >= kEpiWarp0;
    const int q = warp & 3, half = (warp - kEpiWarp0) >> 2, row = q * 32 + lane;
    const uint32_t lane_addr = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    const int GO = WO / 16;   // 16-column groups per owner slice
    auto part_in_range = [&](int j, int p) {   // does CTA j hold a partial of part p?
        const int a0 = j * G / KS, a1 = (j + 1) * G / KS;
        return p == 0 ? a0 < G0 : a1 > G0;
    };
    if (epi) {
        mbar_wait(tfull, 0);
        tc_fence_after();
    }
    __syncwarp();
    tc_fence_before();
    cluster_sync_all();   // (1) all partials final, all stages drained
    tc_fence_after();
    const uint32_t recv = smem_u32(pStage);
    const uint32_t slot_bytes = static_cast<uint32_t>(a.n_parts) * GO * 4u * 128u * 16u;
    if (epi) {
        for (int jj = 1; jj < KS; ++jj) {
            const int j = (rank + jj) % KS;                 // destination owner
            const int slot = rank < j ? rank : rank - 1;    // this CTA's slot in j's buffer
            const uint32_t rbase = mapa_u32(recv + slot * slot_bytes, static_cast<uint32_t>(j));
            for (int p = 0; p < a.n_parts; ++p) {
                if (!part_in_range(rank, p)) continue;
                for (int g = half; g < GO; g += 2) {
                    uint32_t v[16];
                    tmem_ld16(lane_addr + static_cast<uint32_t>(p * NT + j * WO + g * 16), v);
                    tmem_wait_ld();
                    reg_fence16(v);
                    const uint32_t o = rbase + ((static_cast<uint32_t>(p * GO + g) * 4u) * 128u + row) * 16u;
#pragma unroll
                    for (int pc = 0; pc < 4; ++pc)
                        st_cluster_v4(o + pc * 128u * 16u, v[4 * pc], v[4 * pc + 1], v[4 * pc + 2], v[4 * pc + 3]);
                }
            }
        }
    }
    __syncwarp();
    cluster_sync_all();   // (2) every partial slice has arrived

    if (epi) {
        // ===================== owner epilogue: sum in rank order, BN, residual, ReLU ========
        const int RBO = a.rbo, CO_CHUNK = a.co_chunk;
        const int co_shift = CO_CHUNK == 16 ? 4 : (CO_CHUNK == 32 ? 5 : 6);
        const uint32_t row_off = static_cast<uint32_t>(row * RBO);
        const int row_x = (row >> (RBO == 128 ? 0 : (RBO == 64 ? 1 : 2))) & ((RBO >> 4) - 1);
        const bool leader = (warp == kEpiWarp0 && lane == 0);
        const int P = a.Ho * a.Wo;
        if (has_res) mbar_wait(rfull, 0);
        const uint8_t *pRecv = pStage;
        for (int g = half; g < GO; g += 2) {
            float acc[2][16];
#pragma unroll
            for (int p = 0; p < 2; ++p) {
#pragma unroll
                for (int i = 0; i < 16; ++i) acc[p][i] = 0.f;
                if (p >= a.n_parts) continue;
                for (int j = 0; j < KS; ++j) {
                    if (!part_in_range(j, p)) continue;
                    if (j == rank) {
                        uint32_t v[16];
                        tmem_ld16(lane_addr + static_cast<uint32_t>(p * NT + rank * WO + g * 16), v);
                        tmem_wait_ld();
                        reg_fence16(v);
#pragma unroll
                        for (int i = 0; i < 16; ++i) acc[p][i] += __uint_as_float(v[i]);
                    } else {
                        const int slot = j < rank ? j : j - 1;
                        const uint8_t *src =
                            pRecv + slot * slot_bytes + ((static_cast<uint32_t>(p * GO + g) * 4u) * 128u + row) * 16u;
#pragma unroll
                        for (int pc = 0; pc < 4; ++pc) {
                            const float4 f4 = *reinterpret_cast<const float4 *>(src + pc * 128u * 16u);
                            acc[p][4 * pc] += f4.x;
                            acc[p][4 * pc + 1] += f4.y;
                            acc[p][4 * pc + 2] += f4.z;
                            acc[p][4 * pc + 3] += f4.w;
                        }
                    }
                }
            }
            const int cl = g * 16;   // channel inside the owner slice
            float f[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) f[i] = fmaf(acc[0][i], sBN[cl + i], sBN[WO + cl + i]);
            if (a.n_parts > 1) {
#pragma unroll
                for (int i = 0; i < 16; ++i) f[i] += fmaf(acc[1][i], sBN[2 * WO + cl + i], sBN[3 * WO + cl + i]);
            }
            const int oc = cl >> co_shift, q16 = (cl & (CO_CHUNK - 1)) >> 3;
            const uint32_t off0 = oc * oc_bytes + row_off + ((q16 ^ row_x) << 4);
            const uint32_t off1 = oc * oc_bytes + row_off + (((q16 + 1) ^ row_x) << 4);
            if (has_res) {
                const uint4 r0 = *reinterpret_cast<const uint4 *>(pRes + off0);
                const uint4 r1 = *reinterpret_cast<const uint4 *>(pRes + off1);
                const uint32_t rr[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    f[2 * i] += bf16_lo(rr[i]);
                    f[2 * i + 1] += bf16_hi(rr[i]);
                }
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) f[i] = fmaxf(f[i], a.relu_lo);
            if (a.pool_out) {
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    if (o >= P) break;
#pragma unroll
                    for (int i = 0; i < 16; ++i) f[i] += __shfl_xor_sync(0xffffffffu, f[i], o);
                }
                const int n = n0 + row / P;
                if ((lane % P) == 0 && n < a.B) {
                    const float inv = 1.f / static_cast<float>(P);
                    float4 *dst = reinterpret_cast<float4 *>(a.pool_out + static_cast<size_t>(n) * a.c_out + co_own + cl);
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        dst[i] = make_float4(f[4 * i] * inv, f[4 * i + 1] * inv, f[4 * i + 2] * inv, f[4 * i + 3] * inv);
                }
            } else {
                uint32_t o[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) o[i] = pack_bf16(f[2 * i], f[2 * i + 1]);
                *reinterpret_cast<uint4 *>(pOut + off0) = make_uint4(o[0], o[1], o[2], o[3]);
                *reinterpret_cast<uint4 *>(pOut + off1) = make_uint4(o[4], o[5], o[6], o[7]);
            }
        }
        if (!a.pool_out) {
            fence_proxy_async();
            named_bar_sync(1, kEpiThreads);
            if (leader) {
                for (uint32_t j = 0; j < a.n_out_chunks; ++j)
                    tma_store_4d(&tmOut, smem_u32(pOut + j * oc_bytes), co_own + j * a.co_chunk, 0, h0, n0);
                bulk_commit();
                bulk_wait0();
            }
        }
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

size_t conv_splitk_smem_bytes(const SplitArgs &a) {
    const size_t slice = static_cast<size_t>(a.n_out_chunks) * 128 * a.rbo;
    return 1024 + static_cast<size_t>(a.n_stages) * a.stage_bytes + slice * (a.epi == EPI_BN_ADD_RELU ? 2 : 1) +
           16 * static_cast<size_t>(a.w_o) + 8 * (2 * static_cast<size_t>(a.n_stages) + 2) + 16;
}

size_t conv_splitk_recv_bytes(const SplitArgs &a) {
    return static_cast<size_t>(a.ks - 1) * a.n_parts * 128 * a.w_o * 4;
}

cudaError_t launch_conv_splitk(const SplitArgs &a, const CUtensorMap &tmA0, const CUtensorMap &tmB0,
                               const CUtensorMap &tmA1, const CUtensorMap &tmB1, const CUtensorMap &tmRes,
                               const CUtensorMap &tmOut, int grid, cudaStream_t stream, bool pdl) {
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(conv_splitk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kSplitThreads);
    cfg.dynamicSmemBytes = conv_splitk_smem_bytes(a);
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = a.ks;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, conv_splitk_kernel, tmA0, tmB0, tmA1, tmB1, tmRes, tmOut, a);
}

}  // namespace slim
