// kernels_halo.cu -- stride-1 3x3 width-sliced conv on tcgen05 with ONE halo load per
// channel chunk serving all nine filter taps ("kw-split accumulators").
//
// Same operation as conv_umma_kernel (kernels_umma.cu): out = relu(s*conv(x) + t [+ res]),
// the first c_in / c_out channels of the full-width KRSC weights selected by TMA bounds.
// Different data movement, because on B200 the per-tap design is bound by TMA
// issue rate (~28-48 B/cycle/SM for one issuing thread, tools/ubench):
//
//   A: the tile is `rows` whole image rows (rows*W = 128 pixels); its input halo,
//      rows h0-1 .. h0+rows (zero-filled outside the image by TMA), is ONE box
//      [64 ch, W, rows+2, 1].  For tap row kh the UMMA A operand is the contiguous
//      128-row window starting at halo row kh (a descriptor offset of kh*W*128 B).
//   kw: instead of shifting A by one pixel (which breaks the 8-row core-matrix
//      layout at row ends), each kw has its own TMEM accumulator
//          acc_kw[h][w] = sum_kh x[h+kh-1][w] . W[kh][kw]
//      and the epilogue forms out[h][w] = acc_0[h][w-1] + acc_1[h][w] + acc_2[h][w+1]
//      with warp shuffles (W divides 32, so a pixel's W-neighbours are lanes +-1 of
//      the same warp; zero at w = 0 / W-1 is the conv's zero padding).
//   B: the 9 taps x n_tile x 64-channel weight block is one box [64, n_tile, 9]
//      (weight-stationary: loaded once per CTA when all chunks fit in smem), else
//      streamed per (chunk, kh) as [64, n_tile, 3].
//   Small images (H*W < 128, segments 2-3): a tile is tile_imgs = 128/(H*W) whole images and
//      every activation map is addressed as (C, W, N, H) -- image inside row -- so the halo box
//      [64, W, tile_imgs, H+2] lands row-major as (row, image, column): the kh window is again
//      one contiguous 128-row run (offset kh*tile_imgs*W rows), a pixel's W-neighbours are
//      lanes +-1, and the output / residual boxes use the same order (no reshuffle).
// Roles: warp 0 = A producer, warp 1 = MMA issuer, warp 2 = B producer, warp 3 = residual
// prefetch, warps 4..19 = epilogue (four per TMEM lane quarter).
#include "slim_internal.h"
#include "ptx_sm100.cuh"

namespace slim {
using namespace ptx;
namespace {

constexpr int kHaloEpiWarps = 16;   // four per TMEM lane quarter: the epilogue is latency bound
constexpr int kHaloThreads = (4 + kHaloEpiWarps) * 32;   // warps 0 A, 1 MMA, 2 B, 3 residual, 4..19 epilogue
// compact variant (narrow layers): 8 epilogue warps, <= 85 registers, <= ~110 KB smem and <= 256 TMEM
// columns, so two CTAs -- of this kernel or of a concurrent width instance's -- share an SM
constexpr int kHaloThreadsSmall = (4 + 8) * 32;

// kNarrow: runtime channel-chunk geometry (16/32-channel boxes); false folds 64-channel / 128-B rows.
// kVar: 0 = plain / residual epilogue, 1 = + projection shortcut, 2 = + fused average pool,
// 3 = stride-2 conv (parity planes), 4 = three shifted halo boxes (no kw accumulators), see below
// (compile-time, so the common variant carries none of the other two's code)
// kClu: 0 = one CTA per tile (no cluster instructions compiled in: a kernel holding cta_group::2 /
// multicast code must be launched as a cluster), 1 = streamed-weight multicast (a.bmc), 2 = 2-SM pair
// kGN: GroupNorm in the epilogue for layers whose tile covers whole images (segments 2-3):
// pass 1 reduces each (image, 16-channel group)'s statistics from the TMEM-resident fp32 accumulators,
// pass 2 normalises (y*A + Bc, A = rstd*gamma, Bc = beta - mean*A) in place of the BN affine
template <bool kNarrow, int kVar, bool kSmall = false, int kClu = 0, bool kGN = false>
__global__ void __launch_bounds__(kSmall ? kHaloThreadsSmall : kHaloThreads, kSmall ? 2 : 1)
    conv_halo_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmRes, const __grid_constant__ CUtensorMap tmOut,
                     const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmB1,
                     const __grid_constant__ CUtensorMap tmBh, const HaloArgs a) {
    extern __shared__ uint8_t smem_raw[];
    constexpr int EPIW = kSmall ? 8 : kHaloEpiWarps, EPIT = EPIW * 32;   // epilogue warps / threads
    const int CK = kNarrow ? a.ck : kChunk, RBK = kNarrow ? a.rbk : 128;
    const int CO_CHUNK = kNarrow ? a.co_chunk : kChunk, RBO = kNarrow ? a.rbo : 128;
    // 1 KiB alignment without leaving the shared address space (LDS/STS, not generic LD/ST)
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t oc_bytes = 128u * RBO;
    const uint32_t chunk_bytes = a.n_out_chunks * oc_bytes;
    const int n_res = (a.epi == EPI_BN_ADD_RELU) ? a.res_slots : 0;
    const uint32_t sA = smem_u32(smem);
    const uint32_t sB = sA + a.sa * a.a_slot;
    const uint32_t sOut = sB + a.sb * a.b_bytes;
    const int n_grp = a.epi_groups;
    const uint32_t sRes = sOut + n_grp * chunk_bytes;
    uint8_t *pOut = smem + (sOut - sA);
    uint8_t *pRes = smem + (sRes - sA);
    float *sBN = reinterpret_cast<float *>(pRes + n_res * chunk_bytes);
    constexpr bool proj = kVar == 1;   // + 1x1 stride-2 projection shortcut (4th accumulator)
    constexpr bool pool = kVar == 2;   // fused global average pool instead of the store
    // kVar 3: stride-2 conv (block-0 conv1 of segments 1-3).  The input splits into row-parity x
    // column-parity planes, each one TMA box with traversal stride 2: per chunk an "odd-row pair"
    // slot (rows 2h-1, rows+1 of them; odd | even columns) serves kh = 0 and 2 (row offsets 0, 1)
    // and an "even-row pair" slot (rows 2h) serves kh = 1.  kw = 0 and 2 read the odd columns
    // (2w-1 = odd col w-1, 2w+1 = odd col w): one MMA of N = 2n into [acc_kw0 | acc_kw2]; kw = 1
    // reads the even columns: one MMA of N = n into acc_kw1.  Epilogue: acc_kw0[w-1] + acc_kw2[w]
    // + acc_kw1[w].  A traffic = the input once (4x the output tile) instead of 9x.
    constexpr bool s2 = kVar == 3;
    // kVar 4 ("x3"): each chunk's slot holds THREE halo boxes shifted by kw-1 columns (TMA zero-fills
    // the row ends), so every tap is a pure descriptor offset into its box: one accumulator, no
    // shuffles -- for epilogue-bound layers (seg 0, one 64-channel chunk) at 3x the A traffic.
    constexpr bool x3 = kVar == 4;
    // kVar 5 ("x2"): two boxes per chunk -- unshifted (kw = 1 and kw = 2 as one N = 2n MMA into
    // [acc_m | acc_2]) and shifted by -1 column (kw = 0, N = n into acc_m) -- so the epilogue reads
    // two accumulators (acc_m[w] + acc_2[w+1]) instead of three: TMEM reads (~64 B/cycle/SM) are what
    // pace the three-accumulator epilogue of single-chunk layers.
    constexpr bool x2 = kVar == 5;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sBN + (proj ? 4 : 2) * a.c_out);
    const uint32_t bar0 = smem_u32(bars);
    // barriers: a_full[4] a_empty[4] b_full[4] b_empty[4] t_full[4] t_empty[4] r_full[4] r_empty[4]
    // (the B ring has up to kMaxSB slots: the pair variant's half stages are deeper in flight)
    auto a_full = [&](int i) { return bar0 + 8u * i; };
    auto a_empty = [&](int i) { return bar0 + 8u * (4 + i); };
    auto b_full = [&](int i) { return bar0 + 8u * (8 + i); };
    auto b_empty = [&](int i) { return bar0 + 8u * (8 + kMaxSB + i); };
    auto t_full = [&](int i) { return bar0 + 8u * (8 + 2 * kMaxSB + i); };
    auto t_empty = [&](int i) { return bar0 + 8u * (12 + 2 * kMaxSB + i); };
    auto r_full = [&](int i) { return bar0 + 8u * (16 + 2 * kMaxSB + i); };
    auto r_empty = [&](int i) { return bar0 + 8u * (20 + 2 * kMaxSB + i); };
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + kHaloBars);
    // GroupNorm statistics partials (a.gn_part): [tile group][16-ch group of the tile][lane quarter][image]
    float4 *sGN = reinterpret_cast<float4 *>((reinterpret_cast<uintptr_t>(tmem_slot + 4) + 15) & ~uintptr_t(15));
    const int gn_ng = a.n_tile / 16, gn_ni = a.tile_imgs;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int total = a.m_tiles * a.n_tiles;
    // GN image pairs (a.gn_pairs, segment 1: an image is two M tiles): the CTA takes both tiles of an image
    // back to back (its it-th tile is 2u + (it & 1)), so both accumulators are in TMEM for the statistics
    const bool prs = kGN && a.gn_pairs;
    // tile t -> (M tile, N tile): M-fastest by default; a.nfast: N-fastest, so the n_tiles tiles that read
    // the same input rows run at the same time on neighbouring CTAs and the input comes from DRAM once
    // (large batches); pair / image-pair modes keep their two tiles (t, t+1) on consecutive M tiles
    auto decode = [&](int t, int &mt, int &nt) {
        if (!a.nfast) {
            mt = t % a.m_tiles;
            nt = t / a.m_tiles;
        } else if (kClu == 2 || prs) {   // (pair)
            const int u = t >> 1;
            mt = 2 * (u / a.n_tiles) + (t & 1);
            nt = u % a.n_tiles;
        } else {
            mt = t / a.n_tiles;
            nt = t % a.n_tiles;
        }
    };
    auto tile_at = [&](int it) {
        if (!prs) return static_cast<int>(blockIdx.x) + it * static_cast<int>(gridDim.x);
        return 2 * (static_cast<int>(blockIdx.x) + (it >> 1) * static_cast<int>(gridDim.x)) + (it & 1);
    };
    unsigned long long *tr = a.trace ? a.trace + blockIdx.x * 8 : nullptr;
    unsigned long long *td = (a.trace && blockIdx.x == 0) ? a.trace + 2048 : nullptr;   // per-tile detail, CTA 0
#define TD(role, tile, pt) \
    if (td && (tile) < 64) td[(role) * 256 + (tile) * 4 + (pt)] = gtimer()
    if (tr && threadIdx.x == 0) tr[0] = gtimer();
    // 2-SM pair: rank 0 (leader) issues the M = 256 MMAs; the producers of both CTAs signal the leader's
    // full barriers, the leader's commits arrive on both CTAs' empty / t_full barriers, and the peer's
    // accumulator release is relayed onto the leader's t_empty by the peer's (otherwise idle) MMA warp
    constexpr bool pair = kClu == 2;
    const uint32_t prank = pair ? cluster_ctarank() : 0u;
    const bool leader_cta = prank == 0;

    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) {
            mbar_init(a_full(i), 1);
            mbar_init(a_empty(i), 1);
        }
        for (int i = 0; i < kMaxSB; ++i) {
            mbar_init(b_full(i), 1);
            mbar_init(b_empty(i), kClu == 1 ? a.bmc : 1);   // B multicast: every CTA of the cluster frees the slot
        }
        for (int i = 0; i < 4; ++i) {
            mbar_init(t_full(i), 1);
            mbar_init(t_empty(i), EPIT / n_grp + (pair && leader_cta ? 1 : 0));
            mbar_init(r_full(i), 1);
            mbar_init(r_empty(i), EPIT / n_grp);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_tmap(&tmA);
        prefetch_tmap(&tmB);
        prefetch_tmap(&tmOut);
        if (n_res) prefetch_tmap(&tmRes);
    }
    if (warp == 1) {
        if (pair) {   // both CTAs of the pair allocate (same columns): the pair MMA writes both TMEMs
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(a.tmem_cols)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(a.tmem_cols)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
    }
    for (int i = threadIdx.x; i < a.c_out; i += blockDim.x) {
        sBN[i] = a.scale[i];
        sBN[a.c_out + i] = a.shift[i];
        if (proj) {
            sBN[2 * a.c_out + i] = a.scale1[i];
            sBN[3 * a.c_out + i] = a.shift1[i];
        }
    }
    // weight-stationary B does not depend on the previous kernel: start it before the PDL wait
    __syncthreads();
    const int bmc = kClu == 1 ? a.bmc : 1;
    const uint16_t bmask = static_cast<uint16_t>((1u << bmc) - 1u);
    if (kClu != 0) cluster_sync_all();   // every CTA's barriers exist before a peer multicasts / commits into them
    if (a.stationary && warp == 2 && lane == 0) {
        // exact box bytes (the slot itself is rounded up to 1 KiB)
        mbar_expect_tx(b_full(0), static_cast<uint32_t>(a.n_chunks) * 9u * a.n_tile * RBK);
        const uint32_t per_chunk = 9u * a.n_tile * RBK;
        if (!s2) {
            for (int ch = 0; ch < a.n_chunks; ++ch) tma_load_3d(sB + ch * per_chunk, &tmB, b_full(0), ch * CK, 0, 0);
        } else {   // one-tap boxes, per kh in the order kw = 0, 2, 1
            const uint32_t tapb = static_cast<uint32_t>(a.n_tile) * RBK;
            for (int ch = 0; ch < a.n_chunks; ++ch)
                for (int kh = 0; kh < 3; ++kh)
                    for (int j = 0; j < 3; ++j)
                        tma_load_3d(sB + ch * per_chunk + (kh * 3 + j) * tapb, &tmB, b_full(0), ch * CK, 0,
                                    kh * 3 + (j == 0 ? 0 : (j == 1 ? 2 : 1)));
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // the weight producer does not depend on the previous kernel; with flag_in nobody waits for the whole
    // previous grid -- the A / residual producers wait per tile on its flags instead
    if (warp != 2 && !a.flag_in) pdl_wait();
    if (a.flag_zero) {   // later layers' counters (their previous use is complete: we waited for our predecessor)
        if (warp != 2)
            for (int i = blockIdx.x * (blockDim.x - 32) + (threadIdx.x - (warp > 2 ? 32 : 0)); i < a.flag_zero_n;
                 i += gridDim.x * (blockDim.x - 32))
                a.flag_zero[i] = 0u;
        __threadfence();
        __syncthreads();
    }
    pdl_launch_dependents();
    // wait until the previous layer's M tiles that M tile mt reads (its halo rows) are finished
    auto wait_inputs = [&](int mt) {
        if (!a.flag_in) return;
        const int tpi = a.tiles_per_img;
        const int lo = tpi > 1 ? (mt / tpi) * tpi : mt, hi = tpi > 1 ? lo + tpi - 1 : mt;
        // the (up to three) counters are loaded together: one L2 round trip per poll, not three -- the producer
        // issues a tile every ~1.2 us, so serial acquires would make it the bottleneck
        const int m0 = max(lo, mt - 1), m2 = min(hi, mt + 1);
        const uint32_t tgt = static_cast<uint32_t>(a.flag_in_target);
        for (uint32_t spins = 0;; ++spins) {
            // relaxed loads (an acquire load would hold back the next one), then one acquire fence
            const uint32_t f0 = ld_relaxed_gpu(a.flag_in + m0);
            const uint32_t f1 = m0 + 1 <= m2 ? ld_relaxed_gpu(a.flag_in + m0 + 1) : tgt;
            const uint32_t f2 = m0 + 2 <= m2 ? ld_relaxed_gpu(a.flag_in + m0 + 2) : tgt;
            if (f0 >= tgt && f1 >= tgt && f2 >= tgt) {
                fence_acq_rel_gpu();
                break;
            }
            __nanosleep(64);
            if (spins > (1u << 26)) __trap();   // a lost dependency must not hang the GPU
        }
        fence_proxy_async_global();   // the TMA loads that follow see those tiles' TMA stores
    };
    if (tr && threadIdx.x == 0) tr[1] = gtimer();
    const int tiles_per_img = a.tiles_per_img;

    if (warp == 0) {
        // ===================== A producer ============================================
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int ti = 0, t; (t = tile_at(ti)) < total; ++ti) {
                int mt, nt_unused;
                decode(t, mt, nt_unused);
                const int n = mt / tiles_per_img, h0 = (mt - n * tiles_per_img) * a.rows;
                wait_inputs(mt);
                TD(0, ti, 0);
                for (int ch = 0; ch < a.n_chunks && !s2; ++ch) {
                    if (x3 || x2) {   // one slot per kw-shifted box (x2: shifts 0 then -1)
                        for (int kw = 0; kw < (x2 ? 2 : 3); ++kw) {
                            mbar_wait(a_empty(s), ph ^ 1);
                            mbar_expect_tx(a_full(s), a.a_bytes);
                            tma_load_4d(sA + s * a.a_slot, &tmA, a_full(s), ch * CK, x2 ? -kw : kw - 1,
                                        n * a.tile_imgs, h0 - 1);
                            if (kw < (x2 ? 1 : 2) && ++s == a.sa) {
                                s = 0;
                                ph ^= 1;
                            }
                        }
                    } else if (pair) {   // own tile's halo; the leader's a_full counts both CTAs' bytes
                        mbar_wait(a_empty(s), ph ^ 1);
                        const uint32_t lb = mapa_u32(a_full(s), 0);
                        if (leader_cta) mbar_expect_tx(a_full(s), 2u * a.a_bytes);
                        tma_load_4d_pair(sA + s * a.a_slot, &tmA, lb, ch * CK, 0, n * a.tile_imgs, h0 - 1);
                    } else {
                        mbar_wait(a_empty(s), ph ^ 1);
                        if (ch == 0) TD(0, ti, 2);
                        mbar_expect_tx(a_full(s), a.a_bytes);
                        tma_load_4d(sA + s * a.a_slot, &tmA, a_full(s), ch * CK, 0, n * a.tile_imgs, h0 - 1);
                    }
                    if (++s == a.sa) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                for (int ch = 0; ch < a.n_chunks && s2; ++ch) {
                    // odd-row pair (tmA1: rows+1 rows from input row 2h0-1), then even-row pair
                    // (tmA: rows rows from 2h0); each pair = odd-column plane, even-column plane
                    const uint32_t oplane = static_cast<uint32_t>((a.rows + 1) * a.row_px) * RBK;
                    const uint32_t eplane = static_cast<uint32_t>(a.rows * a.row_px) * RBK;
                    mbar_wait(a_empty(s), ph ^ 1);
                    if (pair) {   // own planes; the leader's a_full counts both CTAs' bytes
                        const uint32_t lb = mapa_u32(a_full(s), 0);
                        if (leader_cta) mbar_expect_tx(a_full(s), 4u * oplane);
                        tma_load_4d_pair(sA + s * a.a_slot, &tmA1, lb, ch * CK, 1, n * a.tile_imgs, 2 * h0 - 1);
                        tma_load_4d_pair(sA + s * a.a_slot + oplane, &tmA1, lb, ch * CK, 0, n * a.tile_imgs, 2 * h0 - 1);
                    } else {
                        mbar_expect_tx(a_full(s), 2u * oplane);
                        tma_load_4d(sA + s * a.a_slot, &tmA1, a_full(s), ch * CK, 1, n * a.tile_imgs, 2 * h0 - 1);
                        tma_load_4d(sA + s * a.a_slot + oplane, &tmA1, a_full(s), ch * CK, 0, n * a.tile_imgs, 2 * h0 - 1);
                    }
                    if (++s == a.sa) {
                        s = 0;
                        ph ^= 1;
                    }
                    mbar_wait(a_empty(s), ph ^ 1);
                    if (pair) {
                        const uint32_t lb = mapa_u32(a_full(s), 0);
                        if (leader_cta) mbar_expect_tx(a_full(s), 4u * eplane);
                        tma_load_4d_pair(sA + s * a.a_slot, &tmA, lb, ch * CK, 1, n * a.tile_imgs, 2 * h0);
                        tma_load_4d_pair(sA + s * a.a_slot + eplane, &tmA, lb, ch * CK, 0, n * a.tile_imgs, 2 * h0);
                    } else {
                        mbar_expect_tx(a_full(s), 2u * eplane);
                        tma_load_4d(sA + s * a.a_slot, &tmA, a_full(s), ch * CK, 1, n * a.tile_imgs, 2 * h0);
                        tma_load_4d(sA + s * a.a_slot + eplane, &tmA, a_full(s), ch * CK, 0, n * a.tile_imgs, 2 * h0);
                    }
                    if (++s == a.sa) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                // projection chunks: the stride-2 sampled block input (128 px x 64 ch) and its
                // 1x1 weights (n_tile x 64) share one A slot
                int mt_unused, nt_b;
                decode(t, mt_unused, nt_b);
                const int co0 = nt_b * a.n_tile;
                for (int cp = 0; proj && cp < a.n_chunks_p; ++cp) {
                    mbar_wait(a_empty(s), ph ^ 1);
                    if (pair) {   // own 128 px + HALF of the 1x1 weights (tmB1 box: n_tile/2 rows)
                        const uint32_t lb = mapa_u32(a_full(s), 0);
                        if (leader_cta) mbar_expect_tx(a_full(s), 2u * 16384u + static_cast<uint32_t>(a.n_tile) * 128u);
                        tma_load_4d_pair(sA + s * a.a_slot, &tmA1, lb, cp * kChunk, 0, n * a.tile_imgs, 2 * h0);
                        tma_load_3d_pair(sA + s * a.a_slot + 16384u, &tmB1, lb, cp * kChunk, 0,
                                         co0 + static_cast<int>(prank) * (a.n_tile / 2));
                        if (++s == a.sa) {
                            s = 0;
                            ph ^= 1;
                        }
                        continue;
                    }
                    mbar_expect_tx(a_full(s), 16384u + static_cast<uint32_t>(a.n_tile) * 128u);
                    tma_load_4d(sA + s * a.a_slot, &tmA1, a_full(s), cp * kChunk, 0, n * a.tile_imgs, 2 * h0);
                    tma_load_3d(sA + s * a.a_slot + 16384u, &tmB1, a_full(s), cp * kChunk, 0, co0);
                    if (++s == a.sa) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
            if (tr) tr[2] = gtimer();
        }
    } else if (warp == 3) {
        // ===================== residual prefetch (own warp: never gates the A ring) ===
        if (lane == 0 && n_res) {
            int rs = 0;
            uint32_t rph = 0;
            for (int ti = 0, t; (t = tile_at(ti)) < total; ++ti) {
                int mt, nt;
                decode(t, mt, nt);
                const int n = mt / tiles_per_img, h0 = (mt - n * tiles_per_img) * a.rows, co0 = nt * a.n_tile;
                wait_inputs(mt);   // (the residual is older than the input: transitively finished)
                mbar_wait(r_empty(rs), rph ^ 1);
                TD(0, ti, 1);
                if (a.debug & 8) {
                    mbar_arrive(r_full(rs));
                } else {
                    mbar_expect_tx(r_full(rs), chunk_bytes);
                    for (uint32_t j = 0; j < a.n_out_chunks; ++j)
                        tma_load_4d(sRes + rs * chunk_bytes + j * oc_bytes, &tmRes, r_full(rs), co0 + j * CO_CHUNK, 0,
                                    n * a.tile_imgs, h0);
                }
                if (++rs == n_res) {
                    rs = 0;
                    rph ^= 1;
                }
            }
        }
    } else if (warp == 2) {
        // ===================== B producer (streaming weights) ======================
        if (lane == 0 && !a.stationary) {
            int s = 0;
            uint32_t ph = 0;
            // multicast: this CTA's share of each stage = rows [rank*hrows, +hrows) of every tap block
            const int hrows = a.n_tile / bmc;
            const uint32_t rank = kClu == 1 ? cluster_ctarank() : 0u;
            const uint32_t tapb = static_cast<uint32_t>(a.n_tile) * RBK, hoff = rank * hrows * RBK;
            for (int ti = 0, t; (t = tile_at(ti)) < total; ++ti) {
                int mt_unused, nt_b;
                decode(t, mt_unused, nt_b);
                const int co0 = nt_b * a.n_tile;
                for (int ch = 0; ch < a.n_chunks; ++ch)
                    for (int kq = 0; kq < 3; ++kq) {
                        const int kh = s2 ? (kq == 0 ? 0 : (kq == 1 ? 2 : 1)) : kq;   // s2 consumes kh 0, 2, 1
                        mbar_wait(b_empty(s), ph ^ 1);
                        if (pair) {
                            // the pair MMA's N = 3n rows are ordered [kw0 | kw1 | kw2 of channels 0..n/2) then
                            // [kw0 | kw1 | kw2 of channels n/2..n): this CTA's half is ONE box [ck, n/2, 3 taps]
                            // (the epilogue reads the accumulators in that column order)
                            const uint32_t lb = mapa_u32(b_full(s), 0);
                            if (leader_cta) mbar_expect_tx(b_full(s), 3u * a.n_tile * RBK);
                            if (s2) {   // stride 2: [kw0 | kw2] (N = 2n) split by tap, kw1 (N = n) by channel half:
                                        // this CTA holds tap kw0 (rank 0) or kw2 (rank 1), then its half of kw1
                                tma_load_3d_pair(sB + s * a.b_bytes, &tmB, lb, ch * CK, co0, kh * 3 + (prank ? 2 : 0));
                                tma_load_3d_pair(sB + s * a.b_bytes + static_cast<uint32_t>(a.n_tile) * RBK, &tmBh, lb,
                                                 ch * CK, co0 + static_cast<int>(prank) * (a.n_tile / 2), kh * 3 + 1);
                            } else {
                                tma_load_3d_pair(sB + s * a.b_bytes, &tmBh, lb, ch * CK,
                                                 co0 + static_cast<int>(prank) * (a.n_tile / 2), kh * 3);
                            }
                            if (++s == a.sb) {
                                s = 0;
                                ph ^= 1;
                            }
                            continue;
                        }
                        mbar_expect_tx(b_full(s), 3u * a.n_tile * RBK);   // all bmc shares land in every CTA
                        if (kClu == 1) {   // tap blocks in the consumer's order (s2: kw = 0, 2, 1)
                            for (int j = 0; j < 3; ++j)
                                tma_load_3d_mc(sB + s * a.b_bytes + j * tapb + hoff, &tmBh, b_full(s), ch * CK,
                                               co0 + static_cast<int>(rank) * hrows,
                                               kh * 3 + (s2 ? (j == 0 ? 0 : (j == 1 ? 2 : 1)) : j), bmask);
                        } else if (!s2) {
                            tma_load_3d(sB + s * a.b_bytes, &tmB, b_full(s), ch * CK, co0, kh * 3);
                        } else {   // one-tap boxes in the order kw = 0, 2, 1
                            const uint32_t tapb = static_cast<uint32_t>(a.n_tile) * RBK;
                            tma_load_3d(sB + s * a.b_bytes, &tmB, b_full(s), ch * CK, co0, kh * 3);
                            tma_load_3d(sB + s * a.b_bytes + tapb, &tmB, b_full(s), ch * CK, co0, kh * 3 + 2);
                            tma_load_3d(sB + s * a.b_bytes + 2 * tapb, &tmB, b_full(s), ch * CK, co0, kh * 3 + 1);
                        }
                        if (++s == a.sb) {
                            s = 0;
                            ph ^= 1;
                        }
                    }
            }
        }
    } else if (warp == 1 && pair && !leader_cta) {
        // ===================== pair peer: accumulator-release relay =================
        // the leader's MMA may overwrite an accumulator stage only when BOTH CTAs' epilogues have
        // drained it: forward each completion of this CTA's t_empty(stage) to the leader's
        if (lane == 0) {
            int it = 0;
            for (int t = blockIdx.x; t < total; t += gridDim.x, ++it) {
                const int as = it % a.acc_stages;
                mbar_wait(t_empty(as), static_cast<uint32_t>(it / a.acc_stages) & 1u);
                mbar_arrive_cluster(mapa_u32(t_empty(as), 0));
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer ===========================================
        // Lean issue loop: descriptors are base + offset adds (start-address field, 16-B
        // units), the kh x kw x kk nest has constant trip counts and is fully unrolled --
        // a single issuing thread is otherwise instruction-bound (~120 cycles per MMA,
        // tools/ubench) instead of tensor/smem-bound (~48 cycles at N=64).
        {   // the whole warp runs the loop (uniform operands); one elected lane issues
            // kw_fuse taps per MMA: N = kw_fuse * n_tile covers adjacent accumulators / B tap blocks
            const int kf = a.kw_fuse;
            // pair: M = 256 over the CTA pair; commits arrive on both CTAs' barriers
            auto mma = [&](uint32_t d, uint64_t ad, uint64_t bd, uint32_t id, uint32_t acc) {
                if (pair) umma_bf16_pair(d, ad, bd, id, acc);
                else umma_bf16(d, ad, bd, id, acc);
            };
            auto commit = [&](uint32_t bar) {
                if (pair) umma_commit_pair(bar, 3);
                else umma_commit(bar);
            };
            const int kTileMM = pair ? 2 * kTileM : kTileM;
            const uint32_t idesc = umma_idesc_bf16(kTileMM, a.n_tile * kf);
            const uint32_t idesc_r = umma_idesc_bf16(kTileMM, a.n_tile * (kf == 2 ? 1 : kf));
            const uint32_t tap16 = static_cast<uint32_t>(a.n_tile * RBK) >> 4;   // one tap's B tile, 16-B units
            const uint32_t row16 = static_cast<uint32_t>(a.row_px * RBK) >> 4;   // one halo row (tile_imgs x W px)
            const uint64_t adesc0 = umma_desc_kmajor(sA, RBK), bdesc0 = umma_desc_kmajor(sB, RBK);
            const int kmax = CK >> 4;
            const uint32_t a_slot16 = a.a_slot >> 4, b_slot16 = a.b_bytes >> 4;
            const uint32_t accs = static_cast<uint32_t>(a.acc_stride);
            int s = 0, bs = 0, as = 0;
            uint32_t ph = 0, bph = 0, aph = 0;
            if (a.stationary) {
                mbar_wait(b_full(0), 0);
                tc_fence_after();
            }
            for (int ti = 0, t; (t = tile_at(ti)) < total; ++ti) {
                if (lane == 0) TD(1, ti, 0);
                mbar_wait(t_empty(as), aph ^ 1);
                if (lane == 0) TD(1, ti, 1);
                tc_fence_after();
                const uint32_t acc = tmem_base + static_cast<uint32_t>(as * a.stage_cols);
                if (s2) {
                    const uint32_t idesc2 = umma_idesc_bf16(kTileMM, 2 * a.n_tile), idesc1 = umma_idesc_bf16(kTileMM, a.n_tile);
                    // pair: B of [kw0 | kw2] = this CTA's n rows at the slot start, kw1 = its n/2 rows after them
                    const uint32_t kw1_off16 = pair ? static_cast<uint32_t>(a.n_tile * RBK) >> 4 : 2 * tap16;
                    const uint32_t oplane16 = static_cast<uint32_t>((a.rows + 1) * a.row_px * RBK) >> 4;
                    const uint32_t eplane16 = static_cast<uint32_t>(a.rows * a.row_px * RBK) >> 4;
                    for (int ch = 0; ch < a.n_chunks; ++ch) {
                        const int nk = min(kmax, (a.c_in - ch * CK + 15) >> 4);
                        for (int pr = 0; pr < 2; ++pr) {   // pr 0: odd-row pair (kh 0, 2), pr 1: even-row pair (kh 1)
                            mbar_wait(a_full(s), ph);
                            tc_fence_after();
                            const uint64_t ad = adesc0 + s * a_slot16;
                            const uint32_t plane16 = pr ? eplane16 : oplane16;
                            for (int q = 0; q < (pr ? 1 : 2); ++q) {
                                const int kh = pr ? 1 : 2 * q;
                                const uint32_t roff = (kh == 2) ? row16 : 0u;
                                uint64_t bk;
                                if (a.stationary) {
                                    bk = bdesc0 + static_cast<uint32_t>(ch * 9 + kh * 3) * tap16;
                                } else {
                                    mbar_wait(b_full(bs), bph);
                                    tc_fence_after();
                                    bk = bdesc0 + bs * b_slot16;
                                }
                                if (elect_one() && !(a.debug & 2)) {
                                    for (int kk = 0; kk < nk; ++kk) {
                                        const bool accum = (ch | kh | kk) != 0;
                                        // odd columns -> [acc_kw0 | acc_kw2], even columns -> acc_kw1
                                        mma(acc, ad + roff + 2 * kk, bk + 2 * kk, idesc2, accum);
                                        mma(acc + 2 * accs, ad + plane16 + roff + 2 * kk, bk + kw1_off16 + 2 * kk, idesc1,
                                            accum);
                                    }
                                }
                                __syncwarp();
                                if (!a.stationary) {
                                    if (elect_one()) {
                                        if (kClu == 1) umma_commit_mc(b_empty(bs), bmask);
                                        else commit(b_empty(bs));
                                    }
                                    __syncwarp();
                                    if (++bs == a.sb) {
                                        bs = 0;
                                        bph ^= 1;
                                    }
                                }
                            }
                            if (elect_one()) commit(a_empty(s));
                            __syncwarp();
                            if (++s == a.sa) {
                                s = 0;
                                ph ^= 1;
                            }
                        }
                    }
                }
                for (int ch = 0; ch < a.n_chunks && x3; ++ch) {
                    // x3: one A slot per kw box; weights stationary (host guarantees)
                    const int nk = min(kmax, (a.c_in - ch * CK + 15) >> 4);
                    const uint32_t idesc1 = umma_idesc_bf16(kTileM, a.n_tile);
                    const uint64_t bch = bdesc0 + static_cast<uint32_t>(ch * 9) * tap16;
                    for (int kw = 0; kw < 3; ++kw) {
                        mbar_wait(a_full(s), ph);
                        tc_fence_after();
                        const uint64_t ad = adesc0 + s * a_slot16;
                        if (elect_one() && !(a.debug & 2)) {
#pragma unroll
                            for (int kh = 0; kh < 3; ++kh)
                                for (int kk = 0; kk < nk; ++kk)
                                    umma_bf16(acc, ad + kh * row16 + 2 * kk, bch + (kh * 3 + kw) * tap16 + 2 * kk, idesc1,
                                              (ch | kw | kh | kk) != 0);
                            umma_commit(a_empty(s));
                        }
                        __syncwarp();
                        if (++s == a.sa) {
                            s = 0;
                            ph ^= 1;
                        }
                    }
                }
                for (int ch = 0; ch < a.n_chunks && x2; ++ch) {
                    // x2: slot 0 = unshifted box -> [acc_m | acc_2] (N = 2n, taps kw 1, 2 adjacent in B),
                    //     slot 1 = box shifted -1 -> acc_m (N = n, tap kw 0); weights stationary
                    const int nk = min(kmax, (a.c_in - ch * CK + 15) >> 4);
                    const uint32_t idesc1 = umma_idesc_bf16(kTileM, a.n_tile), idesc2 = umma_idesc_bf16(kTileM, 2 * a.n_tile);
                    const uint64_t bch = bdesc0 + static_cast<uint32_t>(ch * 9) * tap16;
                    for (int bx = 0; bx < 2; ++bx) {
                        mbar_wait(a_full(s), ph);
                        tc_fence_after();
                        const uint64_t ad = adesc0 + s * a_slot16;
                        if (elect_one() && !(a.debug & 2)) {
#pragma unroll
                            for (int kh = 0; kh < 3; ++kh)
                                for (int kk = 0; kk < nk; ++kk) {
                                    if (bx == 0)
                                        umma_bf16(acc, ad + kh * row16 + 2 * kk, bch + (kh * 3 + 1) * tap16 + 2 * kk, idesc2,
                                                  (ch | kh | kk) != 0);
                                    else
                                        umma_bf16(acc, ad + kh * row16 + 2 * kk, bch + (kh * 3) * tap16 + 2 * kk, idesc1, true);
                                }
                            umma_commit(a_empty(s));
                        }
                        __syncwarp();
                        if (++s == a.sa) {
                            s = 0;
                            ph ^= 1;
                        }
                    }
                }
                for (int ch = 0; ch < a.n_chunks && !s2 && !x3 && !x2; ++ch) {
                    const int nk = min(kmax, (a.c_in - ch * CK + 15) >> 4);
                    mbar_wait(a_full(s), ph);
                    if (ch == 0 && lane == 0) TD(1, ti, 2);
                    tc_fence_after();
                    const uint64_t ad = adesc0 + s * a_slot16;
                    if (ch == 0 && lane == 0) TD(3, ti, 0);
                    if (a.stationary) {
                        // one elected issue block for the whole chunk (27 or 36 MMAs, no waits inside)
                        const uint64_t bch = bdesc0 + static_cast<uint32_t>(ch * 9) * tap16;
                        if (elect_one() && !(a.debug & 2)) {
                            if (kf == 3) {
                                // one MMA per (kh, k-step) writes all three kw accumulators
#pragma unroll
                                for (int kh = 0; kh < 3; ++kh)
                                    for (int kk = 0; kk < nk; ++kk)
                                        umma_bf16(acc, ad + kh * row16 + 2 * kk, bch + (kh * 3) * tap16 + 2 * kk, idesc,
                                                  (ch | kh | kk) != 0);
                            } else if (kf == 2) {
#pragma unroll
                                for (int kh = 0; kh < 3; ++kh)
                                    for (int kk = 0; kk < nk; ++kk) {
                                        umma_bf16(acc, ad + kh * row16 + 2 * kk, bch + (kh * 3) * tap16 + 2 * kk, idesc,
                                                  (ch | kh | kk) != 0);
                                        umma_bf16(acc + 2 * accs, ad + kh * row16 + 2 * kk,
                                                  bch + (kh * 3 + 2) * tap16 + 2 * kk, idesc_r, (ch | kh | kk) != 0);
                                    }
                            } else if (nk == 4) {
#pragma unroll
                                for (int kh = 0; kh < 3; ++kh)
#pragma unroll
                                    for (int kw = 0; kw < 3; ++kw)
#pragma unroll
                                        for (int kk = 0; kk < 4; ++kk)
                                            umma_bf16(acc + kw * accs, ad + kh * row16 + 2 * kk,
                                                      bch + (kh * 3 + kw) * tap16 + 2 * kk, idesc, (ch | kh | kk) != 0);
                            } else {
#pragma unroll
                                for (int kh = 0; kh < 3; ++kh)
#pragma unroll
                                    for (int kw = 0; kw < 3; ++kw)
                                        for (int kk = 0; kk < nk; ++kk)
                                            umma_bf16(acc + kw * accs, ad + kh * row16 + 2 * kk,
                                                      bch + (kh * 3 + kw) * tap16 + 2 * kk, idesc, (ch | kh | kk) != 0);
                            }
                        }
                        __syncwarp();
                    } else {
#pragma unroll
                        for (int kh = 0; kh < 3; ++kh) {
                            mbar_wait(b_full(bs), bph);
                            tc_fence_after();
                            const uint64_t bd = bdesc0 + bs * b_slot16;
                            const uint64_t adk = ad + kh * row16;
                            if (elect_one()) {
                                if (!(a.debug & 2)) {
#pragma unroll
                                    for (int kw = 0; kw < 3; kw += kf)
#pragma unroll
                                        for (int kk = 0; kk < 4; ++kk)
                                            if (kk < nk)
                                                mma(acc + kw * accs, adk + 2 * kk, bd + kw * tap16 + 2 * kk,
                                                    kw ? idesc_r : idesc, (ch | kh | kk) != 0);
                                }
                                if (kClu == 1) umma_commit_mc(b_empty(bs), bmask);   // frees the slot cluster-wide
                                else commit(b_empty(bs));
                            }
                            __syncwarp();
                            if (++bs == a.sb) {
                                bs = 0;
                                bph ^= 1;
                            }
                        }
                    }
                    if (ch == 0 && lane == 0) TD(3, ti, 1);
                    if (elect_one()) commit(a_empty(s));
                    __syncwarp();
                    if (ch == 0 && lane == 0) TD(3, ti, 2);
                    if (++s == a.sa) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                if (proj) {
                    const uint32_t idesc_p = umma_idesc_bf16(kTileMM, a.n_tile);
                    const uint64_t pdesc0 = umma_desc_kmajor(sA, 128);
                    for (int cp = 0; cp < a.n_chunks_p; ++cp) {
                        const int nk = min(4, (a.c_in_p - cp * kChunk + 15) >> 4);
                        mbar_wait(a_full(s), ph);
                        tc_fence_after();
                        if (elect_one()) {
                            const uint64_t ad = pdesc0 + s * a_slot16;
                            for (int kk = 0; kk < nk; ++kk)
                                mma(acc + 3 * accs, ad + 2 * kk, ad + (16384u >> 4) + 2 * kk, idesc_p, (cp | kk) != 0);
                            commit(a_empty(s));
                        }
                        __syncwarp();
                        if (++s == a.sa) {
                            s = 0;
                            ph ^= 1;
                        }
                    }
                }
                if (elect_one()) commit(t_full(as));
                __syncwarp();
                if (lane == 0) {
                    TD(1, ti, 3);
                    TD(3, ti, 3);
                }
                if (++as == a.acc_stages) {
                    as = 0;
                    aph ^= 1;
                }
            }
            if (tr && lane == 0) tr[3] = gtimer();
        }
    } else if (warp >= kEpiWarp0) {
        // ===================== epilogue (warps 4..19, four per TMEM lane quarter) ===
        // n_grp (1, 2 or 4) tile groups: group g takes tiles ti = g mod n_grp with accumulator
        // stages, residual slots, a staging buffer and a named barrier of its own, so n_grp tiles'
        // epilogues overlap; inside a group the 4/n_grp warps of a lane quarter split the columns.
        const int q = warp & 3;
        const int quad = (warp - kEpiWarp0) >> 2;          // 0 .. EPIW/4 - 1
        const int cw = (EPIW / 4) / n_grp;                  // column ways per group
        const int grp = quad / cw;
        const int g0 = quad % cw, gstep = cw;
        const int gthreads = EPIT / n_grp;
        const int row = q * 32 + lane;
        // TMA swizzle of the staging tile (rbo-byte rows): 16-B piece q of this row lives at q ^ row_x
        const int co_shift = CO_CHUNK == 16 ? 4 : (CO_CHUNK == 32 ? 5 : 6);
        const uint32_t row_off = static_cast<uint32_t>(row * RBO);
        const int row_x = (row >> (RBO == 128 ? 0 : (RBO == 64 ? 1 : 2))) & ((RBO >> 4) - 1);
        const int w = lane % a.W;                  // W divides 32: pixel column of this row
        const bool leader = (warp == kEpiWarp0 + 4 * cw * grp && lane == 0);
        const uint32_t lane_addr = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
        const float *s0 = sBN, *t0 = sBN + a.c_out;
        const uint32_t sOutG = sOut + grp * chunk_bytes;
        uint8_t *pOutG = pOut + grp * chunk_bytes;
        const float mL = w > 0 ? 1.f : 0.f, mR = w < a.W - 1 ? 1.f : 0.f;   // conv zero padding in W
        // (flag_out) the group's last two tiles: a tile is published once its store has completed, checked when
        // the group's next-but-one tile starts (wait_group 1: never stalls on the store just issued)
        int prev_mt = -1, prev2_mt = -1;
        for (int ti = grp, t; (t = tile_at(ti)) < total; ti += n_grp) {
            int mt, nt;
            decode(t, mt, nt);
            const int n = mt / tiles_per_img, h0 = (mt - n * tiles_per_img) * a.rows, co0 = nt * a.n_tile;
            const int as = ti % a.acc_stages, rs = n_res ? ti % n_res : 0;
            const uint32_t aph = (ti / a.acc_stages) & 1, rph = n_res ? (ti / n_res) & 1 : 0;
            mbar_wait(t_full(as), aph);
            if (leader) TD(2, ti, 0);
            tc_fence_after();
            if (leader && a.flag_out && prev2_mt >= 0) {   // the tile before the previous one: its store is complete
                bulk_wait1();                               // (the previous tile's may still be in flight)
                fence_proxy_async_global();
                red_release_gpu_add(a.flag_out + prev2_mt, 1u);
                prev2_mt = -1;
            }
            if (leader) bulk_wait_read0();   // this group's previous store has left the staging tile
            if (leader) TD(2, ti, 1);
            named_bar_sync(1 + grp, gthreads);
            if (n_res) mbar_wait(r_full(rs), rph);
            if (leader) TD(2, ti, 2);
            const uint8_t *resp = pRes + rs * chunk_bytes;
            const uint32_t col0 = static_cast<uint32_t>(as * a.stage_cols);
            // GN statistics partials of this tile group: [g][tile of the pair][lane quarter][image] (then the
            // projection's); image pairs: the even tile computes them for both tiles (both accumulators are in
            // TMEM: acc_stages == 2), the odd tile reuses them
            const int pm = prs ? 2 : 1;
            float4 *sG = kGN ? sGN + static_cast<size_t>(grp) * gn_ng * pm * 4 * gn_ni * (proj ? 2 : 1) : nullptr;
            if (kGN && !(prs && (ti & 1))) {
                // (K, S1, S2) of this thread's 16 values shifted by K = the image's first lane's first value
                // (keeps the sums of squares from cancelling), summed over the warp's lanes of the same image
                // in a fixed butterfly, parked per (g, quarter, image); merged in pass 2
                auto park = [&](const float (&y)[16], float4 *dst) {
                    const float K = __shfl_sync(0xffffffffu, y[0], ((lane % a.row_px) / a.W) * a.W);
                    const unsigned long long K2 = f2pk(-K, -K);
                    unsigned long long s1 = 0ull, s2q = 0ull;
#pragma unroll
                    for (int i = 0; i < 16; i += 2) {
                        const unsigned long long d = fadd2(f2pk(y[i], y[i + 1]), K2);
                        s1 = fadd2(s1, d);
                        s2q = ffma2(d, d, s2q);
                    }
                    float a1, b1, a2, b2;
                    f2upk(s1, a1, b1);
                    f2upk(s2q, a2, b2);
                    float S1 = a1 + b1, S2 = a2 + b2;
                    for (int ofs = 1; ofs < 32; ofs <<= 1) {
                        if (ofs >= a.W && ofs < a.row_px) continue;   // would mix images of the tile
                        S1 += __shfl_xor_sync(0xffffffffu, S1, ofs);
                        S2 += __shfl_xor_sync(0xffffffffu, S2, ofs);
                    }
                    if (lane < a.row_px && lane % a.W == 0) dst[lane / a.W] = make_float4(K, S1, S2, 0.f);
                };
                if (prs) {   // the image's second tile (next stage) must have landed too
                    mbar_wait(t_full(as + 1), aph);
                    tc_fence_after();
                }
                for (int gi = g0; gi < pm * (a.n_tile / 16); gi += gstep) {
                    const int g = gi % (a.n_tile / 16), h = gi / (a.n_tile / 16);   // h: tile of the pair
                    const uint32_t cs = col0 + static_cast<uint32_t>(h * a.stage_cols);
                    uint32_t v0[16], v1[16], v2[16];
                    tmem_ld16(lane_addr + cs + g * 16, v0);
                    tmem_ld16(lane_addr + cs + a.acc_stride + g * 16, v1);
                    tmem_ld16(lane_addr + cs + 2 * a.acc_stride + g * 16, v2);
                    tmem_wait_ld();
                    reg_fence16(v0);
                    reg_fence16(v1);
                    reg_fence16(v2);
                    float y[16];
                    if (s2) {   // acc_kw0[w-1] + acc_kw2[w] + acc_kw1[w] (as in pass 2)
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const float left = __shfl_up_sync(0xffffffffu, __uint_as_float(v0[i]), 1);
                            y[i] = fmaf(mL, left, __uint_as_float(v1[i]) + __uint_as_float(v2[i]));
                        }
                    } else {
                        const unsigned long long mL2 = f2pk(mL, mL), mR2 = f2pk(mR, mR);
#pragma unroll
                        for (int i = 0; i < 16; i += 2) {
                            const float l0 = __shfl_up_sync(0xffffffffu, __uint_as_float(v0[i]), 1);
                            const float l1 = __shfl_up_sync(0xffffffffu, __uint_as_float(v0[i + 1]), 1);
                            const float r0 = __shfl_down_sync(0xffffffffu, __uint_as_float(v2[i]), 1);
                            const float r1 = __shfl_down_sync(0xffffffffu, __uint_as_float(v2[i + 1]), 1);
                            f2upk(ffma2(mR2, f2pk(r0, r1),
                                        ffma2(mL2, f2pk(l0, l1), f2pk(__uint_as_float(v1[i]), __uint_as_float(v1[i + 1])))),
                                  y[i], y[i + 1]);
                        }
                    }
                    park(y, sG + ((g * pm + h) * 4 + q) * gn_ni);
                    if (proj) {   // the projection shortcut's own GroupNorm statistics
                        tmem_ld16(lane_addr + cs + 3 * a.acc_stride + g * 16, v0);
                        tmem_wait_ld();
                        reg_fence16(v0);
#pragma unroll
                        for (int i = 0; i < 16; ++i) y[i] = __uint_as_float(v0[i]);
                        park(y, sG + (((gn_ng + g) * pm + h) * 4 + q) * gn_ni);
                    }
                }
                named_bar_sync(1 + grp, gthreads);
            }
            // GN: (mean, rstd) of this thread's image for 16-channel group g from the four quarter partials
            // (equal counts, fixed merge order: bitwise batch independent); base = the layer's or projection's
            auto gn_stats = [&](int g, int base) {
                const float4 *pq = sG + ((base + g) * pm * 4) * gn_ni + (lane % a.row_px) / a.W;
                const float cq = 16.f * 32.f * static_cast<float>(a.W) / static_cast<float>(a.row_px);
                auto quarter = [&](const float4 v) {
                    const float m = v.y / cq;
                    return make_float2(v.x + m, fmaf(-v.y, m, v.z));
                };
                auto merge = [](float2 x, float2 y2, float c) {
                    const float d = y2.x - x.x;
                    return make_float2((x.x + y2.x) * 0.5f, (x.y + y2.y) + d * d * (c * 0.5f));
                };
                auto four = [&](const float4 *p4) {
                    return merge(merge(quarter(p4[0]), quarter(p4[gn_ni]), cq),
                                 merge(quarter(p4[2 * gn_ni]), quarter(p4[3 * gn_ni]), cq), 2.f * cq);
                };
                float2 tot = four(pq);
                if (prs) tot = merge(tot, four(pq + 4 * gn_ni), 4.f * cq);   // the image's two tiles
                return make_float2(tot.x, rsqrtf(tot.y / (4.f * pm * cq) + a.gn_eps));
            };
            for (int g = g0; g < a.n_tile / 16 && !(a.debug & 16); g += gstep) {
                uint32_t v0[16], v1[16], v2[16];
                // kw accumulator columns of channels g*16..: pair mode interleaves the two channel halves
                // ([kw0 kw1 kw2] of the first n/2 channels, then of the second), else kw * acc_stride + channel
                // (stride 2: each of its two MMAs splits N in natural order -- columns as in the one-CTA kernel)
                constexpr bool ilv = pair && !s2;
                const int hn = ilv ? a.n_tile / 2 : a.acc_stride;
                const uint32_t cb = col0 + static_cast<uint32_t>(ilv ? (g * 16 / hn) * 3 * hn + (g * 16) % hn : g * 16);
                tmem_ld16(lane_addr + cb, v0);
                if (x2) tmem_ld16(lane_addr + col0 + a.acc_stride + g * 16, v2);   // acc_m, acc_2
                if (!x3 && !x2) {
                    tmem_ld16(lane_addr + cb + hn, v1);
                    tmem_ld16(lane_addr + cb + 2 * hn, v2);
                }
                tmem_wait_ld();
                reg_fence16(v0);
                if (x2) reg_fence16(v2);
                if (!x3 && !x2) {
                    reg_fence16(v1);
                    reg_fence16(v2);
                }
                const int cl = g * 16, cg = co0 + cl;
                float f[16];
                // BN: per-channel scale / shift from smem; GN: per (image, channel) A = rstd*gamma, Bc = beta - mean*A
                float gA[kGN ? 16 : 1], gB[kGN ? 16 : 1];
                if constexpr (kGN) {
                    const float2 ms = gn_stats(g, 0);
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        gA[i] = ms.y * s0[cg + i];
                        gB[i] = fmaf(-ms.x, gA[i], t0[cg + i]);
                    }
                }
                auto SC = [&](int i) { if constexpr (kGN) return make_float2(gA[i], gA[i + 1]); else return *reinterpret_cast<const float2 *>(s0 + cg + i); };
                auto SH = [&](int i) { if constexpr (kGN) return make_float2(gB[i], gB[i + 1]); else return *reinterpret_cast<const float2 *>(t0 + cg + i); };
                if (x2) {   // out[w] = acc_m[w] + acc_2[w+1], then BN (packed fp32x2)
                    const unsigned long long mR2 = f2pk(mR, mR);
#pragma unroll
                    for (int i = 0; i < 16; i += 2) {
                        const float r0 = __shfl_down_sync(0xffffffffu, __uint_as_float(v2[i]), 1);
                        const float r1 = __shfl_down_sync(0xffffffffu, __uint_as_float(v2[i + 1]), 1);
                        const unsigned long long y =
                            ffma2(mR2, f2pk(r0, r1), f2pk(__uint_as_float(v0[i]), __uint_as_float(v0[i + 1])));
                        const float2 sc = *reinterpret_cast<const float2 *>(s0 + cg + i);
                        const float2 sh = *reinterpret_cast<const float2 *>(t0 + cg + i);
                        f2upk(ffma2(y, f2pk(sc.x, sc.y), f2pk(sh.x, sh.y)), f[i], f[i + 1]);
                    }
                }
                if (!x3 && !s2 && !x2) {
                    // out[w] = acc_0[w-1] + acc_1[w] + acc_2[w+1] (zero padding at the row ends), then BN:
                    // packed fp32x2 FMAs (per-lane rounding identical to the scalar form)
                    const unsigned long long mL2 = f2pk(mL, mL), mR2 = f2pk(mR, mR);
#pragma unroll
                    for (int i = 0; i < 16; i += 2) {
                        const float l0 = __shfl_up_sync(0xffffffffu, __uint_as_float(v0[i]), 1);
                        const float l1 = __shfl_up_sync(0xffffffffu, __uint_as_float(v0[i + 1]), 1);
                        const float r0 = __shfl_down_sync(0xffffffffu, __uint_as_float(v2[i]), 1);
                        const float r1 = __shfl_down_sync(0xffffffffu, __uint_as_float(v2[i + 1]), 1);
                        const unsigned long long y = ffma2(
                            mR2, f2pk(r0, r1), ffma2(mL2, f2pk(l0, l1), f2pk(__uint_as_float(v1[i]), __uint_as_float(v1[i + 1]))));
                        const float2 sc = SC(i);
                        const float2 sh = SH(i);
                        f2upk(ffma2(y, f2pk(sc.x, sc.y), f2pk(sh.x, sh.y)), f[i], f[i + 1]);
                    }
                }
#pragma unroll
                for (int i = 0; i < 16 && (x3 || s2); ++i) {
                    float y;
                    if (x3) {
                        f[i] = fmaf(__uint_as_float(v0[i]), s0[cg + i], t0[cg + i]);
                        continue;
                    }
                    const float left = __shfl_up_sync(0xffffffffu, __uint_as_float(v0[i]), 1);
                    if (s2) {   // acc_kw0[w-1] + acc_kw2[w] + acc_kw1[w]
                        y = fmaf(mL, left, __uint_as_float(v1[i]) + __uint_as_float(v2[i]));
                    } else {
                        const float right = __shfl_down_sync(0xffffffffu, __uint_as_float(v2[i]), 1);
                        y = fmaf(mR, right, fmaf(mL, left, __uint_as_float(v1[i])));
                    }
                    if constexpr (kGN) f[i] = fmaf(y, gA[i], gB[i]);
                    else f[i] = fmaf(y, s0[cg + i], t0[cg + i]);
                }
                if (proj) {   // + s_sc * proj + t_sc (the shortcut's own BN)
                    tmem_ld16(lane_addr + col0 + 3 * a.acc_stride + g * 16, v0);
                    tmem_wait_ld();
                    reg_fence16(v0);
                    const float *s1 = sBN + 2 * a.c_out, *t1 = sBN + 3 * a.c_out;
                    if constexpr (kGN) {   // the shortcut's GroupNorm: its own statistics, gamma / beta
                        const float2 ms = gn_stats(g, gn_ng);
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            gA[i] = ms.y * s1[cg + i];
                            gB[i] = fmaf(-ms.x, gA[i], t1[cg + i]);
                        }
                    }
#pragma unroll
                    for (int i = 0; i < 16; i += 2) {   // f + (s1 * p + t1), pairwise packed
                        const float2 sc = kGN ? SC(i) : *reinterpret_cast<const float2 *>(s1 + cg + i);
                        const float2 sh = kGN ? SH(i) : *reinterpret_cast<const float2 *>(t1 + cg + i);
                        const unsigned long long pr =
                            ffma2(f2pk(__uint_as_float(v0[i]), __uint_as_float(v0[i + 1])), f2pk(sc.x, sc.y),
                                  f2pk(sh.x, sh.y));
                        f2upk(fadd2(f2pk(f[i], f[i + 1]), pr), f[i], f[i + 1]);
                    }
                }
                const int oc = cl >> co_shift, q16 = (cl & (CO_CHUNK - 1)) >> 3;
                const uint32_t off0 = oc * oc_bytes + row_off + ((q16 ^ row_x) << 4);
                const uint32_t off1 = oc * oc_bytes + row_off + (((q16 + 1) ^ row_x) << 4);
                if (n_res) {
                    const uint4 r0 = *reinterpret_cast<const uint4 *>(resp + off0);
                    const uint4 r1 = *reinterpret_cast<const uint4 *>(resp + off1);
                    const uint32_t rr[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        f2upk(fadd2(f2pk(f[2 * i], f[2 * i + 1]), f2pk(bf16_lo(rr[i]), bf16_hi(rr[i]))), f[2 * i],
                              f[2 * i + 1]);
                }
                if (pool) {
                    // fused global average pool (last conv): sum the W pixels of this image row
                    // (lanes of one image are W consecutive lanes), park it per (row = lane quarter,
                    // image, channel) in the staging tile; rows are summed below in fixed order
#pragma unroll
                    for (int i = 0; i < 16; ++i) f[i] = fmaxf(f[i], a.relu_lo);
                    for (int o = 1; o < a.W; o <<= 1) {
#pragma unroll
                        for (int i = 0; i < 16; ++i) f[i] += __shfl_xor_sync(0xffffffffu, f[i], o);
                    }
                    if (w == 0) {
                        float4 *dst = reinterpret_cast<float4 *>(
                            pOutG + 4u * ((q * a.tile_imgs + lane / a.W) * a.n_tile + cl));
#pragma unroll
                        for (int i = 0; i < 4; ++i) dst[i] = make_float4(f[4 * i], f[4 * i + 1], f[4 * i + 2], f[4 * i + 3]);
                    }
                    continue;
                }
                uint32_t o[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) o[i] = pack_bf16(fmaxf(f[2 * i], a.relu_lo), fmaxf(f[2 * i + 1], a.relu_lo));
                *reinterpret_cast<uint4 *>(pOutG + off0) = make_uint4(o[0], o[1], o[2], o[3]);
                *reinterpret_cast<uint4 *>(pOutG + off1) = make_uint4(o[4], o[5], o[6], o[7]);
                if (a.gn_part) {
                    // GN statistics of the stored values: this thread's 16 (one pixel, one 16-channel group),
                    // shifted by K = lane 0's first value (a sample of the same layer: keeps the sums of
                    // squares from cancelling), summed over the lanes of the same image (fixed butterfly),
                    // parked per (quarter, image) with K; the quarters are merged below
                    // (the image's first lane in this warp: the statistics of an image never depend on
                    // which slot of the tile it occupies -> bitwise batch independent)
                    const float K = __shfl_sync(0xffffffffu, bf16_lo(o[0]), ((lane % a.row_px) / a.W) * a.W);
                    const unsigned long long K2 = f2pk(-K, -K);
                    unsigned long long s1 = 0ull, s2 = 0ull;
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const unsigned long long d = fadd2(f2pk(bf16_lo(o[i]), bf16_hi(o[i])), K2);
                        s1 = fadd2(s1, d);
                        s2 = ffma2(d, d, s2);
                    }
                    float a1, b1, a2, b2;
                    f2upk(s1, a1, b1);
                    f2upk(s2, a2, b2);
                    float S1 = a1 + b1, S2 = a2 + b2;
                    for (int ofs = 1; ofs < 32; ofs <<= 1) {
                        if (ofs >= a.W && ofs < a.row_px) continue;   // would mix images of the tile
                        S1 += __shfl_xor_sync(0xffffffffu, S1, ofs);
                        S2 += __shfl_xor_sync(0xffffffffu, S2, ofs);
                    }
                    if (lane < a.row_px && lane % a.W == 0)
                        sGN[((grp * gn_ng + g) * 4 + q) * gn_ni + lane / a.W] = make_float4(K, S1, S2, 0.f);
                }
            }
            tc_fence_before();
            mbar_arrive(t_empty(as));
            if (n_res) mbar_arrive(r_empty(rs));
            if (pool) {
                named_bar_sync(1 + grp, gthreads);
                const int tig = ((quad - grp * cw) * 4 + q) * 32 + lane;
                const float inv = 1.f / static_cast<float>(a.rows * a.W);
                const float *sp = reinterpret_cast<const float *>(pOutG);
                const int per_row = a.tile_imgs * a.n_tile;
                for (int idx = tig; idx < per_row; idx += gthreads) {
                    const int im = idx / a.n_tile, c = idx - im * a.n_tile;
                    float sum = 0.f;
                    for (int h = 0; h < a.rows; ++h) sum += sp[h * per_row + idx];
                    const int nimg = n * a.tile_imgs + im;
                    if (nimg < a.B) a.pool_out[static_cast<size_t>(nimg) * a.c_out + co0 + c] = sum * inv;
                }
                named_bar_sync(1 + grp, gthreads);   // the parked sums may be overwritten by the next tile
                continue;
            }
            fence_proxy_async();
            named_bar_sync(1 + grp, gthreads);
            if (a.gn_part) {   // merge the four lane quarters (equal counts, fixed order) -> global
                const int tig = ((quad - grp * cw) * 4 + q) * 32 + lane;
                const int ni_tile = a.tile_imgs;
                for (int idx = tig; idx < gn_ng * ni_tile; idx += gthreads) {
                    const int gg = idx / ni_tile, im = idx - gg * ni_tile;
                    const float4 *pq = sGN + ((grp * gn_ng + gg) * 4) * gn_ni + im;
                    const float cq = 16.f * 32.f * static_cast<float>(a.W) / static_cast<float>(a.row_px);   // per partial
                    auto quarter = [&](const float4 v) {   // (K, S1, S2) -> (mean, M2) over cq values
                        const float m = v.y / cq;
                        return make_float2(v.x + m, fmaf(-v.y, m, v.z));
                    };
                    auto merge = [](float2 x, float2 y, float c) {   // two partials of c values each
                        const float d = y.x - x.x;
                        return make_float2((x.x + y.x) * 0.5f, (x.y + y.y) + d * d * (c * 0.5f));
                    };
                    const float2 tot = merge(merge(quarter(pq[0]), quarter(pq[gn_ni]), cq),
                                             merge(quarter(pq[2 * gn_ni]), quarter(pq[3 * gn_ni]), cq), 2.f * cq);
                    int nimg, ti;
                    if (ni_tile == 1) {
                        nimg = mt / tiles_per_img;
                        ti = mt - nimg * tiles_per_img;
                    } else {
                        nimg = mt * ni_tile + im;
                        ti = 0;
                    }
                    if (nimg < a.B) a.gn_part[(static_cast<size_t>(nimg) * tiles_per_img + ti) * (a.c_out / 16) + co0 / 16 + gg] = tot;
                }
            }
            if (leader && !(a.debug & 4)) {
                TD(2, ti, 3);
                for (uint32_t j = 0; j < a.n_out_chunks; ++j)
                    tma_store_4d(&tmOut, sOutG + j * oc_bytes, co0 + j * CO_CHUNK, 0, n * a.tile_imgs, h0);
                bulk_commit();
            }
            prev2_mt = prev_mt;
            prev_mt = mt;
        }
        if (tr && leader) tr[4] = gtimer();
        if (leader) bulk_wait0();
        if (leader && a.flag_out) {
            fence_proxy_async_global();
            if (prev2_mt >= 0) red_release_gpu_add(a.flag_out + prev2_mt, 1u);
            if (prev_mt >= 0) red_release_gpu_add(a.flag_out + prev_mt, 1u);
        }
        if (tr && leader) tr[5] = gtimer();
    }

    tc_fence_before();
    __syncthreads();
    if (kClu != 0) cluster_sync_all();   // no CTA leaves while a peer may still multicast / commit into it
    if (warp == 1) {
        tc_fence_after();
        if (pair)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(a.tmem_cols)
                         : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(a.tmem_cols)
                         : "memory");
    }
    if (tr && threadIdx.x == 0) tr[6] = gtimer();
}

}  // namespace

size_t conv_halo_smem_bytes(const HaloArgs &a) {
    const size_t chunk = static_cast<size_t>(a.n_out_chunks) * 128 * a.rbo;
    const int n_res = (a.epi == EPI_BN_ADD_RELU) ? a.res_slots : 0;
    return 1024 + static_cast<size_t>(a.sa) * a.a_slot + static_cast<size_t>(a.sb) * a.b_bytes +
           chunk * (a.epi_groups + n_res) +
           (a.epi == EPI_BN_PROJ_RELU ? 16 : 8) * static_cast<size_t>(a.c_out) + 8 * kHaloBars + 16 +
           (a.gn_fuse ? static_cast<size_t>(a.epi_groups) * (a.n_tile / 16) * 4 * a.tile_imgs * 16 *
                            (a.epi == EPI_BN_PROJ_RELU ? 2 : 1) * (a.gn_pairs ? 2 : 1) + 16
                      : 0) +
           (a.gn_part ? static_cast<size_t>(a.epi_groups) * (a.n_tile / 16) * 4 * a.tile_imgs * 16 + 16 : 0);
}

cudaError_t launch_conv_halo(const HaloArgs &a, const CUtensorMap &tmA, const CUtensorMap &tmB,
                             const CUtensorMap &tmRes, const CUtensorMap &tmOut, const CUtensorMap &tmA1,
                             const CUtensorMap &tmB1, const CUtensorMap &tmBh, int grid, cudaStream_t stream, bool pdl) {
    using Fn = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap,
                        HaloArgs);
    static const Fn fns[2][6] = {{conv_halo_kernel<false, 0>, conv_halo_kernel<false, 1>, conv_halo_kernel<false, 2>,
                                  conv_halo_kernel<false, 3>, conv_halo_kernel<false, 4>, conv_halo_kernel<false, 5>},
                                 {conv_halo_kernel<true, 0>, conv_halo_kernel<true, 1>, conv_halo_kernel<true, 2>,
                                  conv_halo_kernel<true, 3>, conv_halo_kernel<true, 4>, conv_halo_kernel<true, 5>}};
    static const Fn small_fns[4] = {conv_halo_kernel<true, 0, true>, conv_halo_kernel<true, 1, true>,
                                    conv_halo_kernel<true, 2, true>, conv_halo_kernel<true, 3, true>};
    // cluster variants (streamed weights only: 64-channel boxes, plain / projection / pool / stride 2)
    static const Fn mc_fns[4] = {conv_halo_kernel<false, 0, false, 1>, conv_halo_kernel<false, 1, false, 1>,
                                 conv_halo_kernel<false, 2, false, 1>, conv_halo_kernel<false, 3, false, 1>};
    static const Fn pair_fns[4] = {conv_halo_kernel<false, 0, false, 2>, conv_halo_kernel<false, 1, false, 2>,
                                   conv_halo_kernel<false, 2, false, 2>, conv_halo_kernel<false, 3, false, 2>};
    // GroupNorm in the epilogue (whole-image tiles): plain / projection / pool / stride 2
    static const Fn gn_fns[2][4] = {{conv_halo_kernel<false, 0, false, 0, true>, conv_halo_kernel<false, 1, false, 0, true>,
                                     conv_halo_kernel<false, 2, false, 0, true>, conv_halo_kernel<false, 3, false, 0, true>},
                                    {conv_halo_kernel<true, 0, false, 0, true>, conv_halo_kernel<true, 1, false, 0, true>,
                                     conv_halo_kernel<true, 2, false, 0, true>, conv_halo_kernel<true, 3, false, 0, true>}};
    static bool attr_set = false;
    if (!attr_set) {
        auto big = [](Fn f) {
            cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
            cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
            return e;
        };
        for (int m = 0; m < 2; ++m)
            for (int v = 0; v < 6; ++v)
                if (cudaError_t e = big(fns[m][v]); e != cudaSuccess) return e;
        for (int v = 0; v < 4; ++v)
            if (cudaError_t e = big(mc_fns[v]); e != cudaSuccess) return e;
        for (int v = 0; v < 4; ++v)
            if (cudaError_t e = big(pair_fns[v]); e != cudaSuccess) return e;
        for (int m = 0; m < 2; ++m)
            for (int v = 0; v < 4; ++v)
                if (cudaError_t e = big(gn_fns[m][v]); e != cudaSuccess) return e;
        for (int v = 0; v < 4; ++v) {
            cudaError_t e = cudaFuncSetAttribute(small_fns[v], cudaFuncAttributeMaxDynamicSharedMemorySize, 113 * 1024);
            if (e != cudaSuccess) return e;
            cudaFuncSetAttribute(small_fns[v], cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        }
        attr_set = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(a.small ? kHaloThreadsSmall : kHaloThreads);
    cfg.dynamicSmemBytes = conv_halo_smem_bytes(a);
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = a.pair ? 2 : a.bmc;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (a.bmc > 1 || a.pair) ? 2 : 1;
    if (a.bmc > 1 && (grid % a.bmc || a.m_tiles % a.bmc || a.stationary || a.small)) return cudaErrorInvalidValue;
    if (a.pair && (grid % 2 || a.m_tiles % 2 || a.stationary || a.small || a.bmc > 1 || a.kw_fuse != 3 || a.x3 ||
                   a.n_tile % 16))
        return cudaErrorInvalidValue;
    const bool narrow = a.ck != kChunk || a.co_chunk != kChunk;
    const int var = a.stride2 ? 3 : (a.x3 == 1 ? 4 : (a.x3 == 2 ? 5 : (a.epi == EPI_BN_PROJ_RELU ? 1 : (a.pool_out ? 2 : 0))));
    if (a.small) {
        if (var > 3 || a.bmc > 1 || a.pair) return cudaErrorInvalidValue;
        return cudaLaunchKernelEx(&cfg, small_fns[var], tmA, tmB, tmRes, tmOut, tmA1, tmB1, tmBh, a);
    }
    if (a.gn_fuse) {
        if (var > 3 || a.pair || a.bmc > 1 || a.tiles_per_img != (a.gn_pairs ? 2 : 1) || a.kw_fuse != 3 || a.gn_part ||
            (a.gn_pairs && (a.acc_stages != 2 || a.epi_groups != 1 || grid * 2 > a.m_tiles * a.n_tiles)))
            return cudaErrorInvalidValue;
        return cudaLaunchKernelEx(&cfg, gn_fns[narrow ? 1 : 0][var], tmA, tmB, tmRes, tmOut, tmA1, tmB1, tmBh, a);
    }
    if (a.pair) {
        if (narrow || var > 3) return cudaErrorInvalidValue;
        return cudaLaunchKernelEx(&cfg, pair_fns[var], tmA, tmB, tmRes, tmOut, tmA1, tmB1, tmBh, a);
    }
    if (a.bmc > 1) {
        if (narrow || var > 3) return cudaErrorInvalidValue;
        return cudaLaunchKernelEx(&cfg, mc_fns[var], tmA, tmB, tmRes, tmOut, tmA1, tmB1, tmBh, a);
    }
    return cudaLaunchKernelEx(&cfg, fns[narrow ? 1 : 0][var], tmA, tmB, tmRes, tmOut, tmA1, tmB1, tmBh, a);
}

}  // namespace slim
