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
#include "ptx_sm100.cuh"

#include <cuda_bf16.h>

#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>

namespace slim {
using namespace ptx;
namespace {

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

// Tile sequence of this CTA.  mc == 1: tiles blockIdx.x, +gridDim.x, ... over m_tiles x n_tiles.
// mc > 1: cluster c walks M tiles c, c + n_clusters, ...; CTA rank j of the cluster takes N tiles
// j, j + mc, ... of that M tile, so all CTAs of a cluster run the same k-block sequence in lockstep.
struct TileSeq {
    int start, step, total, rank;
};
__device__ __forceinline__ TileSeq tile_seq(const ConvArgs &a, int mc) {
    TileSeq q;
    if (mc == 1) {
        q.start = blockIdx.x;
        q.step = gridDim.x;
        q.total = a.m_tiles * a.n_tiles;
        q.rank = 0;
    } else {
        q.rank = static_cast<int>(blockIdx.x) % mc;
        q.start = static_cast<int>(blockIdx.x) / mc;
        q.step = static_cast<int>(gridDim.x) / mc;
        q.total = a.m_tiles * (a.n_tiles / mc);
    }
    return q;
}
__device__ __forceinline__ int seq_tile(const ConvArgs &a, const TileSeq &q, int v, int mc) {
    if (mc == 1) return v;
    const int mt = v % a.m_tiles, nn = v / a.m_tiles;
    return (nn * mc + q.rank) * a.m_tiles + mt;
}

// kMode bit 0: cluster multicast of A (a.mc > 1); bit 1: narrow boxes (runtime ck / rbk /
// co_chunk).  Mode 0 folds every layout constant (64-channel chunks, 128-B rows, no cluster).
template <int kMode>
__global__ void __launch_bounds__(kConvThreads, 1)
    conv_umma_kernel(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmB0,
                     const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmB1,
                     const __grid_constant__ CUtensorMap tmRes, const __grid_constant__ CUtensorMap tmOut,
                     const ConvArgs a) {
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment: SW128 TMA boxes and UMMA descriptors (base_offset = 0)
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr bool kMC = (kMode & 1) != 0, kNarrow = (kMode & 2) != 0;
    const int MC = kMC ? a.mc : 1;
    const int RBO = kNarrow ? a.rbo : 128, CO_CHUNK = kNarrow ? a.co_chunk : kChunk;
    const uint32_t A_TILE = kNarrow ? a.a_tile_bytes : static_cast<uint32_t>(kTileABytes);
    const int S = a.n_stages;
    const uint32_t oc_bytes = 128u * RBO;                  // one staging chunk: 128 pixels x co_chunk
    const uint32_t chunk_bytes = a.n_out_chunks * oc_bytes;  // one 128-pixel x n_tile tile
    const uint32_t sA = smem_u32(smem);
    const uint32_t sB = sA + S * A_TILE;
    const uint32_t sOut = sB + S * a.stage_b_bytes;
    const uint32_t sRes = sOut + chunk_bytes;
    const int n_res = (a.epi == EPI_BN_ADD_RELU) ? a.res_slots : 0;
    uint8_t *pOut = smem + (sOut - sA);
    uint8_t *pRes = smem + (sRes - sA);
    float *sBN = reinterpret_cast<float *>(pRes + n_res * chunk_bytes);   // scale0|shift0|scale1|shift1, c_out each
    uint64_t *bars = reinterpret_cast<uint64_t *>(sBN + 4 * a.c_out);
    const uint32_t bar0 = smem_u32(bars);
    // barrier map: full[0,S) empty[S,2S) tmem_full[2S,2S+2) tmem_empty[2S+2,2S+4) res_full[2S+4,+2) res_empty[2S+6,+2)
    auto full_bar = [&](int i) { return bar0 + 8u * i; };
    auto empty_bar = [&](int i) { return bar0 + 8u * (S + i); };
    auto tfull_bar = [&](int i) { return bar0 + 8u * (2 * S + i); };
    auto tempty_bar = [&](int i) { return bar0 + 8u * (2 * S + 2 + i); };
    auto rfull_bar = [&](int i) { return bar0 + 8u * (2 * S + 4 + i); };
    auto rempty_bar = [&](int i) { return bar0 + 8u * (2 * S + 6 + i); };
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * S + 8);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const TileSeq tq = tile_seq(a, MC);
    const uint16_t mc_mask = static_cast<uint16_t>((1u << MC) - 1);
    unsigned long long *tr = a.trace ? a.trace + blockIdx.x * 8 : nullptr;
    // aggregate wait times per CTA (register accumulators, one store per role at the end)
    unsigned long long *tw = a.trace ? a.trace + 2048 + blockIdx.x * 8 : nullptr;
    unsigned long long acc_w0 = 0, acc_w1 = 0;
    if (tr && threadIdx.x == 0) tr[0] = gtimer();

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(full_bar(i), 1);        // the owning producer's arrive.expect_tx (A + B bytes)
            mbar_init(empty_bar(i), MC);    // the MMA commit of every CTA of the cluster
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(tfull_bar(i), 1);
            mbar_init(tempty_bar(i), kEpiThreads);
            mbar_init(rfull_bar(i), 1);
            mbar_init(rempty_bar(i), kEpiThreads);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_tmap(&tmA0);
        prefetch_tmap(&tmB0);
        if (a.n_parts > 1) {
            prefetch_tmap(&tmA1);
            prefetch_tmap(&tmB1);
        }
        if (!a.pool_out) prefetch_tmap(&tmOut);
        if (a.epi == EPI_BN_ADD_RELU) prefetch_tmap(&tmRes);
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(a.tmem_cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    // the folded BN vectors are weights (not produced by the previous kernel): stage
    // them in smem before the PDL wait so the epilogue never waits on global loads
    for (int i = threadIdx.x; i < a.c_out; i += blockDim.x) {
        sBN[i] = a.scale0[i];
        sBN[a.c_out + i] = a.shift0[i];
        if (a.n_parts > 1) {
            sBN[2 * a.c_out + i] = a.scale1[i];
            sBN[3 * a.c_out + i] = a.shift1[i];
        }
    }
    // PDL: everything above overlapped the previous kernel's tail; wait for its
    // results to be visible before any dependent global read, then let the next
    // kernel start its own prologue as SMs free up.
    tc_fence_before();
    __syncthreads();
    if (kMC) cluster_sync_all();   // every CTA's barriers exist before anyone multicasts into them
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // (every producer loads activations, so every warp waits -- griddepcontrol.wait is per thread)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (tr && threadIdx.x == 0) tr[1] = gtimer();

    if (warp == 0 || warp == 2 || warp == 12 || warp == 13) {
        // ============ TMA producers: n_prod warps, k-block kb owned by warp kb % n_prod ============
        // One thread issues at most ~1 TMA per ~500 cycles (tools/ubench: throughput scales with
        // issuing threads, not box bytes), so A+B loads are spread over up to four issuing warps.
        const int pi = warp == 0 ? 0 : (warp == 2 ? 1 : (warp == 12 ? 2 : 3));
        if (lane == 0 && pi < a.n_prod) {
            int stage = 0;
            uint32_t phase = 0;
            uint32_t kb_g = 0;   // k-block counter: producer ownership and the multicast issuer rotate on it
            for (int v = tq.start; v < tq.total; v += tq.step) {
                const TileCoord tc = tile_coord(a, seq_tile(a, tq, v, MC));
                for (int p = 0; p < a.n_parts; ++p) {
                    const GemmPart &gp = a.part[p];
                    const int GP_CK = kNarrow ? gp.ck : kChunk, GP_RBK = kNarrow ? gp.rbk : 128;
                    const CUtensorMap *tA = p ? &tmA1 : &tmA0;
                    const CUtensorMap *tB = p ? &tmB1 : &tmB0;
                    for (int kb = 0; kb < gp.n_kblocks; ++kb) {
                        if (static_cast<int>(kb_g % a.n_prod) == pi) {
                            const int tap = kb / gp.n_chunks, ch = kb - tap * gp.n_chunks;
                            const int kh = tap / gp.ksize, kw = tap - kh * gp.ksize;
                            {
                                const unsigned long long w0 = tw ? gtimer() : 0;
                                mbar_wait(empty_bar(stage), phase ^ 1);
                                if (tw) acc_w0 += gtimer() - w0;
                            }
                            if (a.debug & 1) {
                                mbar_arrive(full_bar(stage));
                            } else {
                                const uint32_t b_bytes = static_cast<uint32_t>(a.n_tile) * GP_RBK;
                                mbar_expect_tx(full_bar(stage), 128u * GP_RBK + b_bytes);
                                const int ah = tc.h0 * gp.stride + kh - gp.pad;
                                if (!kMC)
                                    tma_load_4d(sA + stage * A_TILE, tA, full_bar(stage), ch * GP_CK, kw - gp.pad, ah,
                                                tc.n0);
                                else if (static_cast<int>(kb_g % MC) == tq.rank)
                                    tma_load_4d_mc(sA + stage * A_TILE, tA, full_bar(stage), ch * GP_CK, kw - gp.pad, ah,
                                                   tc.n0, mc_mask);
                                tma_load_3d(sB + stage * a.stage_b_bytes, tB, full_bar(stage), ch * GP_CK, tap, tc.co0);
                            }
                        }
                        if (++stage == S) {
                            stage = 0;
                            phase ^= 1;
                        }
                        ++kb_g;
                    }
                }
            }
            if (tr && warp == 0) tr[2] = gtimer();
            if (tw && pi < 2) tw[pi] = acc_w0;
        }
    } else if (warp == 3) {
        // ===================== residual prefetch (own warp: never gates the A/B ring) =========
        if (lane == 0 && n_res) {
            int rs = 0;
            uint32_t rphase = 0;
            for (int v = tq.start; v < tq.total; v += tq.step) {
                const TileCoord tc = tile_coord(a, seq_tile(a, tq, v, MC));
                mbar_wait(rempty_bar(rs), rphase ^ 1);
                if (a.debug & 8) {
                    mbar_arrive(rfull_bar(rs));
                } else {
                    mbar_expect_tx(rfull_bar(rs), chunk_bytes);
                    for (uint32_t j = 0; j < a.n_out_chunks; ++j)
                        tma_load_4d(sRes + rs * chunk_bytes + j * oc_bytes, &tmRes, rfull_bar(rs), tc.co0 + j * CO_CHUNK, 0,
                                    tc.h0, tc.n0);
                }
                if (++rs == n_res) {
                    rs = 0;
                    rphase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (one thread) =======================
        // lean loop: descriptor = base + offset adds, K-steps unrolled (see kernels_halo.cu)
        {   // whole warp runs the loop (uniform operands), one elected lane issues
            const uint32_t idesc = umma_idesc_bf16(kTileM, a.n_tile);
            const uint32_t a16 = A_TILE >> 4, b16 = a.stage_b_bytes >> 4;
            int stage = 0, as = 0;
            uint32_t phase = 0, aphase = 0;
            for (int v = tq.start; v < tq.total; v += tq.step) {
                {
                    const unsigned long long w0 = tw ? gtimer() : 0;
                    mbar_wait(tempty_bar(as), aphase ^ 1);
                    if (tw) acc_w1 += gtimer() - w0;
                }
                tc_fence_after();
                for (int p = 0; p < a.n_parts; ++p) {
                    const GemmPart &gp = a.part[p];
                    const int GP_CK = kNarrow ? gp.ck : kChunk, GP_RBK = kNarrow ? gp.rbk : 128;
                    const uint32_t d = tmem_base + static_cast<uint32_t>((as * a.n_parts + p) * a.acc_stride);
                    const uint64_t adesc0 = umma_desc_kmajor(sA, GP_RBK), bdesc0 = umma_desc_kmajor(sB, GP_RBK);
                    const int kmax = GP_CK >> 4;
                    const int nchunks = gp.n_chunks;
                    int ch = 0;
                    for (int kb = 0; kb < gp.n_kblocks; ++kb) {
                        const int nk = min(kmax, (gp.c_in - ch * GP_CK + 15) >> 4);
                        {
                            const unsigned long long w0 = tw ? gtimer() : 0;
                            mbar_wait(full_bar(stage), phase);
                            if (tw) acc_w0 += gtimer() - w0;
                        }
                        tc_fence_after();
                        const uint64_t ad = adesc0 + stage * a16;
                        const uint64_t bd = bdesc0 + stage * b16;
                        if (elect_one()) {
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk)   // K=16 per MMA = 32 bytes inside the 128-B atom
                                if (kk < nk && !(a.debug & 2))
                                    umma_bf16(d, ad + 2 * kk, bd + 2 * kk, idesc, (kb | kk) != 0);
                            // frees the smem slot (in every CTA of the cluster) when these MMAs finish
                            if (!kMC) umma_commit(empty_bar(stage));
                            else umma_commit_mc(empty_bar(stage), mc_mask);
                        }
                        __syncwarp();
                        if (++stage == S) {
                            stage = 0;
                            phase ^= 1;
                        }
                        if (++ch == nchunks) ch = 0;
                    }
                }
                if (elect_one()) umma_commit(tfull_bar(as));   // accumulator ready for the epilogue
                __syncwarp();
                if (++as == a.acc_stages) {
                    as = 0;
                    aphase ^= 1;
                }
            }
            if (tr && lane == 0) tr[3] = gtimer();
            if (tw && lane == 0) {
                tw[2] = acc_w0;
                tw[3] = acc_w1;
            }
        }
    } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + 8) {
        // ===================== epilogue (warps 4..11) ========================
        // two warps per TMEM lane quarter; warp half h takes column groups h, h+2, ...
        const int q = warp & 3;              // TMEM lane quarter this warp may access
        const int half = (warp - kEpiWarp0) >> 2;
        const int row = q * 32 + lane;       // pixel row inside the 128-pixel tile
        // TMA swizzle of the staging tile (rbo-byte rows): 16-B piece q of this row lives at q ^ row_x
        const int co_shift = CO_CHUNK == 16 ? 4 : (CO_CHUNK == 32 ? 5 : 6);
        const uint32_t row_off = static_cast<uint32_t>(row * RBO);
        const int row_x = (row >> (RBO == 128 ? 0 : (RBO == 64 ? 1 : 2))) & ((RBO >> 4) - 1);
        const bool leader = (warp == kEpiWarp0 && lane == 0);
        const uint32_t lane_addr = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
        const float *s0 = sBN, *t0 = sBN + a.c_out, *s1 = sBN + 2 * a.c_out, *t1 = sBN + 3 * a.c_out;
        // fused pool: the image of this row and its pixel count P (P divides 32)
        const int P = a.Ho * a.Wo;
        int as = 0, rs = 0;
        uint32_t aphase = 0, rphase = 0;
        for (int v = tq.start; v < tq.total; v += tq.step) {
            const TileCoord tc = tile_coord(a, seq_tile(a, tq, v, MC));
            {
                const unsigned long long w0 = tw ? gtimer() : 0;
                mbar_wait(tfull_bar(as), aphase);
                if (tw) acc_w0 += gtimer() - w0;
            }
            tc_fence_after();
            if (!a.pool_out) {
                if (leader) bulk_wait_read0();   // previous tile's stores have left the staging buffer
                named_bar_sync(1, kEpiThreads);
            }
            if (n_res) mbar_wait(rfull_bar(rs), rphase);
            const uint8_t *resp = pRes + rs * chunk_bytes;
            const uint32_t col0 = static_cast<uint32_t>(as * a.n_parts * a.acc_stride);
            for (int g = half; g < a.n_tile / 16; g += 2) {
                uint32_t v[16], u[16];
                tmem_ld16(lane_addr + col0 + g * 16, v);
                if (a.epi == EPI_BN_PROJ_RELU) tmem_ld16(lane_addr + col0 + a.acc_stride + g * 16, u);
                tmem_wait_ld();
                const int cl = g * 16;             // channel inside the tile
                const int cg = tc.co0 + cl;        // global output channel
                float f[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) f[i] = fmaf(__uint_as_float(v[i]), s0[cg + i], t0[cg + i]);
                if (a.epi == EPI_BN_PROJ_RELU) {
#pragma unroll
                    for (int i = 0; i < 16; ++i) f[i] += fmaf(__uint_as_float(u[i]), s1[cg + i], t1[cg + i]);
                }
                // 16-B pieces q16 and q16+1 of row `row` in staging chunk cl/co_chunk (TMA-swizzled)
                const int oc = cl >> co_shift, q16 = (cl & (CO_CHUNK - 1)) >> 3;
                const uint32_t off0 = oc * oc_bytes + row_off + ((q16 ^ row_x) << 4);
                const uint32_t off1 = oc * oc_bytes + row_off + (((q16 + 1) ^ row_x) << 4);
                if (n_res) {
                    const uint4 r0 = *reinterpret_cast<const uint4 *>(resp + off0);
                    const uint4 r1 = *reinterpret_cast<const uint4 *>(resp + off1);
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
                    // rows of one image are P consecutive lanes (P | 32): butterfly over them
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        if (o >= P) break;
#pragma unroll
                        for (int i = 0; i < 16; ++i) f[i] += __shfl_xor_sync(0xffffffffu, f[i], o);
                    }
                    const int n = tc.n0 + row / P;
                    if ((lane % P) == 0 && n < a.B) {
                        const float inv = 1.f / static_cast<float>(P);
                        float4 *dst = reinterpret_cast<float4 *>(a.pool_out + static_cast<size_t>(n) * a.c_out + cg);
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
            tc_fence_before();
            mbar_arrive(tempty_bar(as));     // TMEM accumulator may be overwritten
            if (n_res) {
                mbar_arrive(rempty_bar(rs));  // residual slot may be refilled
                if (++rs == n_res) {
                    rs = 0;
                    rphase ^= 1;
                }
            }
            if (!a.pool_out) {
                fence_proxy_async();          // generic smem writes -> visible to the TMA (async proxy)
                named_bar_sync(1, kEpiThreads);
                if (leader && !(a.debug & 4)) {
                    for (uint32_t j = 0; j < a.n_out_chunks; ++j)
                        tma_store_4d(&tmOut, sOut + j * oc_bytes, tc.co0 + j * CO_CHUNK, 0, tc.h0, tc.n0);
                    bulk_commit();
                }
            }
            if (++as == a.acc_stages) {
                as = 0;
                aphase ^= 1;
            }
        }
        if (tr && leader) tr[4] = gtimer();
        if (tw && leader) tw[4] = acc_w0;
        if (leader) bulk_wait0();
        if (tr && leader) tr[5] = gtimer();
    }

    tc_fence_before();
    __syncthreads();
    if (kMC) cluster_sync_all();   // no CTA leaves while a peer may still multicast into it
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(a.tmem_cols)
                     : "memory");
    }
    if (tr && threadIdx.x == 0) tr[6] = gtimer();
}

}  // namespace

size_t conv_umma_smem_bytes(const ConvArgs &a) {
    const size_t chunk = static_cast<size_t>(a.n_out_chunks) * 128 * a.rbo;
    const int n_res = (a.epi == EPI_BN_ADD_RELU) ? a.res_slots : 0;
    return 1024 /*alignment slack*/ + static_cast<size_t>(a.n_stages) * (a.a_tile_bytes + a.stage_b_bytes) +
           chunk * (1 + n_res) + 16 * static_cast<size_t>(a.c_out) + 8 * (2 * a.n_stages + 8) + 16;
}

int conv_umma_max_ctas_per_sm(size_t smem_bytes) {
    // cached per shared-memory size: the occupancy query costs microseconds of host time
    static std::mutex mu;
    static std::map<size_t, int> cache;
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(smem_bytes);
    if (it != cache.end()) return it->second;
    int n = 0;
    cudaFuncSetAttribute(conv_umma_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(conv_umma_kernel<0>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, conv_umma_kernel<0>, kConvThreads, smem_bytes) != cudaSuccess) {
        cudaGetLastError();
        n = 1;
    }
    n = n < 1 ? 1 : n;
    cache[smem_bytes] = n;
    return n;
}

namespace {
typedef void (*ConvKernelFn)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, ConvArgs);
ConvKernelFn conv_kernel_for(int mode) {
    switch (mode) {
        case 1: return conv_umma_kernel<1>;
        case 2: return conv_umma_kernel<2>;
        case 3: return conv_umma_kernel<3>;
        default: return conv_umma_kernel<0>;
    }
}
}  // namespace

cudaError_t launch_conv_umma(const ConvArgs &a, const CUtensorMap &tmA0, const CUtensorMap &tmB0,
                             const CUtensorMap &tmA1, const CUtensorMap &tmB1, const CUtensorMap &tmRes,
                             const CUtensorMap &tmOut, int grid, cudaStream_t stream, bool pdl) {
    static bool attr_set = false;
    if (!attr_set) {
        for (int m = 0; m < 4; ++m) {
            cudaError_t e = cudaFuncSetAttribute(conv_kernel_for(m), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 227 * 1024);
            if (e != cudaSuccess) return e;
            cudaFuncSetAttribute(conv_kernel_for(m), cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        }
        attr_set = true;
    }
    // layout constants fold away in mode 0 (all chunks 64 channels / 128-B rows, no cluster)
    bool narrow = a.co_chunk != kChunk || a.part[0].ck != kChunk || (a.n_parts > 1 && a.part[1].ck != kChunk);
    const int mode = (a.mc > 1 ? 1 : 0) | (narrow ? 2 : 0);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kConvThreads);
    cfg.dynamicSmemBytes = conv_umma_smem_bytes(a);
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = a.mc;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = a.mc > 1 ? 2 : 1;   // cluster launch only when multicasting
    return cudaLaunchKernelEx(&cfg, conv_kernel_for(mode), tmA0, tmB0, tmA1, tmB1, tmRes, tmOut, a);
}

}  // namespace slim
