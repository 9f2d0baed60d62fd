// kernels_fused.cu -- segment 0 (stem + two BasicBlocks) as ONE kernel for the
// narrow widths (c0 = 16 | 32 channels, r = 0.25 | 0.5 of C0 = 64), every activation resident in
// shared memory.
//
// Why: at c0 <= 32 each of segment 0's five layers is a few tiny MMAs per 128-pixel tile; as five
// kernels the layer chain is paced by per-launch latency (grid drain, prologue, TMA load -> MMA ->
// epilogue -> TMA store -> next launch), not by bytes or FLOPs (r=0.25 at 0.14 of its
// per-layer roofline, B <= 32 flat at 84-130 us per chain).  Here one CTA takes one whole image
// (32x32 pixels = 8 tiles of 4 rows) through all five layers: the epilogue of layer l writes its
// bf16 output straight into the SW32/SW64 K-major layout the tensor core reads as layer l+1's A
// operand, so a layer boundary is one CTA barrier, not a kernel boundary.
//
// Same arithmetic as the per-layer path (stem_kernel + conv_halo_kernel), bit for bit: the same
// MMAs in the same K order (stem: K = 27 zero-padded to 32 in two K=16 steps; 3x3 convs: kh outer,
// 16-channel K steps inner, the three kw taps fused into one N = 3*c0 MMA into three adjacent TMEM
// accumulators, combined in the epilogue as acc0[w-1] + acc1[w] + acc2[w+1]), the same fp32 epilogue
// operations in the same order, one RNE bf16 rounding per stored value.
//
// Shared memory (1 KiB aligned), RB = 2*c0 bytes per pixel row:
//   X, T   activations with one zero row above and below the image: 34 x 32 pixel rows x RB
//          (the kh = 0 / 2 taps of the first / last image row read the zero rows)
//   Wc     the four convs' weights, [layer][kh][kw][c0 rows][RB], K-major, swizzled
//   Ws     stem weights, c0 rows x 64 B (K = 32), SW64
//   IMG    the image, 32 x 32 x 3 bf16 (6 KiB)
//   the stem's im2col A tiles (4 x 8 KiB, SW64) live inside T between its zero rows
// Warps 0..15: im2col builders and epilogue, group g = warp/4 takes tiles g and g+4, TMEM lane quarter
// q = warp%4 (image row 4t+q, pixel column = lane); warp 16: TMEM owner + MMA issuer.
#include "slim_internal.h"
#include "ptx_sm100.cuh"

namespace slim {
using namespace ptx;
namespace {

constexpr int kFsEpiWarps = 16;
constexpr int kFsThreads = (kFsEpiWarps + 1) * 32;
constexpr int kFsImg = 32;                  // H = W = 32 (CIFAR-shaped input)
constexpr int kFsTiles = 8;                 // 1024 pixels / 128
constexpr int kFsImgBytes = kFsImg * kFsImg * 3 * 2;

__device__ __forceinline__ uint32_t fs_mapa(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void fs_st_cluster(uint32_t addr, uint4 v) {
    asm volatile("st.shared::cluster.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}

// P CTAs per image (a cluster): CTA p owns image rows [4*TPC*p, 4*TPC*(p+1)), TPC = 8/P tiles of 4 rows;
// its activation buffers hold those rows plus one halo row above and below (LR = 4*TPC + 2 rows): at the
// image border the zero padding, inside the image the neighbour CTA's boundary row, which the neighbour's
// epilogue writes there through DSMEM before the layer barrier (P = 1: the whole image, 34 rows).
struct FsLayout {
    uint32_t rb, act, x, t, wc, ws, img, sa, bn, bars, gn, total;
};
__host__ __device__ inline FsLayout fs_layout(int c0, int P) {
    FsLayout L;
    const uint32_t tpc = 8u / P, lr = 4u * tpc + 2u;
    L.rb = 2u * c0;
    L.act = (lr * 32u * L.rb + 1023u) & ~1023u;
    L.x = 0;
    L.t = L.x + L.act;
    L.wc = L.t + L.act;
    L.ws = (L.wc + 4u * 9u * c0 * L.rb + 1023u) & ~1023u;
    L.img = L.ws + ((static_cast<uint32_t>(c0) * 64u + 1023u) & ~1023u);
    // stem im2col A slots (8 KiB each): inside T between its halo rows when T is large enough (P = 1)
    const uint32_t slots = tpc < 4 ? tpc : 4;
    L.sa = (P == 1) ? L.t + 32u * L.rb : ((L.img + kFsImgBytes + 1023u) & ~1023u);
    L.bn = (P == 1) ? L.img + kFsImgBytes : L.sa + slots * 8192u;
    L.bars = L.bn + 5u * 2u * 32u * 4u;
    L.gn = (L.bars + 2u * kFsTiles * 8u + 16u + 15u) & ~15u;   // GroupNorm: partials + coefficients
    L.total = L.gn + 1024u + 256u;
    return L;
}

template <int C0, int P, bool GN>
__global__ void __launch_bounds__(kFsThreads, 1) seg0_fused_kernel(const FusedSeg0Args a) {
    constexpr int RB = 2 * C0, NG = C0 / 16;                 // row bytes, 16-channel groups
    constexpr int SC = C0 == 16 ? 64 : 128;                  // TMEM columns per tile stage (>= 3*C0)
    constexpr int S = 512 / SC;                              // stages: 8 | 4
    constexpr int PCS = RB / 16;                             // 16-B pieces per pixel row
    constexpr int TPC = kFsTiles / P, LR = 4 * TPC + 2;      // tiles / local rows per CTA
    constexpr int ROUND = TPC < 4 ? TPC : 4;                 // stem tiles per round (A slots)
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const FsLayout Lo = fs_layout(C0, P);
    uint8_t *pX = smem + Lo.x, *pT = smem + Lo.t, *pWc = smem + Lo.wc, *pWs = smem + Lo.ws;
    uint8_t *pImg = smem + Lo.img, *pA = smem + Lo.sa;
    float *sBN = reinterpret_cast<float *>(smem + Lo.bn);   // [layer 0..4][scale 32 | shift 32]
    const uint32_t bar0 = smem_u32(smem + Lo.bars);
    auto t_full = [&](int s) { return bar0 + 8u * s; };
    auto t_empty = [&](int s) { return bar0 + 8u * (kFsTiles + s); };
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + Lo.bars + 2 * kFsTiles * 8);
    const uint32_t sX = smem_u32(pX), sT = smem_u32(pT), sWc = smem_u32(pWc), sWs = smem_u32(pWs);
    const uint32_t sA = smem_u32(pA);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = P > 1 ? cluster_ctarank() : 0;
    const int h_base = 4 * TPC * static_cast<int>(rank);   // first image row of this CTA
    // diagnostics: CTA 0, thread 0 (epilogue warp 0) stamps [0..15], the MMA warp's lane 0 [16..31]
    unsigned long long *tr = (a.trace && blockIdx.x == 0) ? a.trace : nullptr;
    int ntr = 0, ntm = 16;
#define FS_STAMP()                                     \
    do {                                               \
        if (tr && tid == 0 && ntr < 16) tr[ntr++] = gtimer(); \
        if (tr && warp == kFsEpiWarps && lane == 0 && ntm < 32) tr[ntm++] = gtimer(); \
    } while (0)
    FS_STAMP();
    // layer barrier: the CTA, or the whole cluster (halo rows written into the neighbours)
    auto layer_sync = [&]() {
        if (P > 1) {
            asm volatile("fence.proxy.async.shared::cluster;" ::: "memory");
            tc_fence_before();
            cluster_sync_all();
        } else {
            fence_proxy_async();
            tc_fence_before();
            __syncthreads();
        }
        tc_fence_after();
    };

    // ---- prologue: nothing here is produced by the previous kernel (before the PDL wait)
    for (int i = tid; i < 32 * RB / 16; i += kFsThreads) {   // zero rows at the image border (never written)
        const uint4 z = make_uint4(0, 0, 0, 0);
        if (rank == 0) {
            reinterpret_cast<uint4 *>(pX)[i] = z;
            reinterpret_cast<uint4 *>(pT)[i] = z;
        }
        if (rank == P - 1) {
            reinterpret_cast<uint4 *>(pX + (LR - 1) * 32 * RB)[i] = z;
            reinterpret_cast<uint4 *>(pT + (LR - 1) * 32 * RB)[i] = z;
        }
    }
    // conv weights: row (l*9 + tap)*C0 + co holds w_l[co][tap][0..C0) (K-major, swizzled); all of a thread's
    // loads are issued before its stores (one global round trip instead of one per piece)
    {
        constexpr int NP = 4 * 9 * C0 * PCS, PER = (NP + kFsThreads - 1) / kFsThreads;
        uint4 v[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int i = tid + k * kFsThreads;
            const int j = i % PCS, row = i / PCS;
            const int co = row % C0, lt = row / C0, tap = lt % 9, l = lt / 9;
            if (i < NP)
                v[k] = *reinterpret_cast<const uint4 *>(a.w[l] + (static_cast<size_t>(co) * 9 + tap) * a.cin_full + j * 8);
        }
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int i = tid + k * kFsThreads;
            if (i < NP) *reinterpret_cast<uint4 *>(pWc + swz_off(i / PCS, i % PCS, RB)) = v[k];
        }
    }
    // stem weights: the SW128 B image built at load (128-B rows, K = 64 padded) -> SW64 rows (K = 32)
    for (int i = tid; i < C0 * 4; i += kFsThreads) {
        const int co = i >> 2, j = i & 3;
        const uint4 v = *reinterpret_cast<const uint4 *>(static_cast<const uint8_t *>(a.stem_b) + co * 128 +
                                                         ((j ^ (co & 7)) << 4));
        *reinterpret_cast<uint4 *>(pWs + swz_off(co, j, 64)) = v;
    }
    for (int i = tid; i < 5 * C0; i += kFsThreads) {
        const int l = i / C0, c = i % C0;
        sBN[l * 64 + c] = a.scale[l][c];
        sBN[l * 64 + 32 + c] = a.shift[l][c];
    }
    if (tid == 0) {
        for (int s = 0; s < kFsTiles; ++s) {
            mbar_init(t_full(s), 1);
            mbar_init(t_empty(s), 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kFsEpiWarps) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    fence_proxy_async();   // generic-proxy weight / zero-row writes -> visible to the tensor core
    tc_fence_before();
    if (P > 1)
        cluster_sync_all();
    else
        __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    FS_STAMP();
    pdl_wait();            // the images may be the previous kernel's output
    pdl_launch_dependents();
    FS_STAMP();

    const int g = warp >> 2, q = warp & 3;                   // epilogue tile group, TMEM lane quarter
    const int row = q * 32 + lane;                           // tile row = local tile row q, column = lane
    const uint32_t lane_addr = tmem + (static_cast<uint32_t>(q * 32) << 16);
    const float mL = lane > 0 ? 1.f : 0.f, mR = lane < 31 ? 1.f : 0.f;   // conv zero padding in W
    uint32_t u = 0;                                          // tile counter: stage u % S, phase u / S
    // an output of local tile t, quarter q: local buffer row lr = 4t + q + 1; the boundary rows also go to
    // the neighbour's halo row (DSMEM)
    auto store_act = [&](uint8_t *buf, int t, int piece, uint4 v) {
        const int lr = 4 * t + q + 1;
        const uint32_t off = static_cast<uint32_t>(buf - smem) + swz_off(lr * 32 + lane, piece, RB);
        *reinterpret_cast<uint4 *>(smem + off) = v;
        if (P > 1) {
            if (lr == 1 && rank > 0)   // first row -> the upper neighbour's bottom halo row
                fs_st_cluster(fs_mapa(smem_u32(smem) + static_cast<uint32_t>(buf - smem) +
                                          swz_off((LR - 1) * 32 + lane, piece, RB), rank - 1), v);
            if (lr == LR - 2 && rank < P - 1)   // last row -> the lower neighbour's top halo row
                fs_st_cluster(fs_mapa(smem_u32(smem) + static_cast<uint32_t>(buf - smem) + swz_off(lane, piece, RB),
                                      rank + 1),
                              v);
        }
    };

    // GroupNorm (GN): two passes per layer over the same (recomputed) accumulators -- pass 1 the per-(image,
    // 16-channel group) statistics of the fp32 raw output (per thread (mean, M2) of its 16 values, merged
    // with equal counts in one fixed tree: 32 lanes -> 4 lane quarters -> tiles; a cluster merges its CTAs'
    // tile partials in the same tree, so P = 1 and P = 8 agree bit for bit), pass 2 the normalisation
    // y * A + Bc (A = rstd * gamma, Bc = beta - mean * A) in the epilogue that BatchNorm uses.
    float2 *sPart = reinterpret_cast<float2 *>(smem + Lo.gn);          // [tile][quarter][group] (count 512)
    float2 *sClu = sPart + kFsTiles * 4 * NG;                           // [rank][group] tile partials (P > 1)
    float *sCoef = reinterpret_cast<float *>(sClu + 8 * NG);            // [A 32 | Bc 32]
    auto merge2 = [](float2 x, float2 y, float c) {   // two partials of c values each
        const float d = y.x - x.x;
        return make_float2((x.x + y.x) * 0.5f, (x.y + y.y) + d * d * (c * 0.5f));
    };
    // per-thread statistics of 16 values, merged over the warp (all 32 lanes: one image row, one group)
    auto warp_stats = [&](const float (&y)[16], int t, int gi) {
        float mu = 0.f;
#pragma unroll
        for (int i = 0; i < 16; ++i) mu += y[i];
        mu *= (1.f / 16.f);
        float m2 = 0.f;
#pragma unroll
        for (int i = 0; i < 16; ++i) m2 = fmaf(y[i] - mu, y[i] - mu, m2);
        float cnt = 16.f;
        for (int ofs = 1; ofs < 32; ofs <<= 1) {
            const float mo = __shfl_xor_sync(0xffffffffu, mu, ofs), qo = __shfl_xor_sync(0xffffffffu, m2, ofs);
            const float d = mo - mu;
            m2 = (m2 + qo) + d * d * (cnt * 0.5f);
            mu = (mu + mo) * 0.5f;
            cnt *= 2.f;
        }
        if (lane == 0) sPart[(t * 4 + q) * NG + gi] = make_float2(mu, m2);
    };
    // after pass 1: the image's statistics per group -> coefficients (layer lgn's gamma / beta in sBN)
    auto gn_finish = [&](int lgn) {
        __syncthreads();
        if (tid < NG) {
            float2 tp[TPC];
#pragma unroll
            for (int t = 0; t < TPC; ++t) {
                const float2 *pq = sPart + (t * 4) * NG + tid;
                tp[t] = merge2(merge2(pq[0], pq[NG], 512.f), merge2(pq[2 * NG], pq[3 * NG], 512.f), 1024.f);
            }
            if (P > 1) {   // this CTA's tile partial into every CTA's rank slot
                for (int pr = 0; pr < P; ++pr)
                    asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(fs_mapa(
                                     smem_u32(sClu + static_cast<int>(rank) * NG + tid), pr)),
                                 "f"(tp[0].x), "f"(tp[0].y)
                                 : "memory");
            } else {
#pragma unroll
                for (int t = 0; t < TPC; ++t) sClu[t * NG + tid] = tp[t];
            }
        }
        if (P > 1) cluster_sync_all();
        else __syncthreads();
        if (tid < NG) {   // fixed pairwise tree over the 8 tile partials (2048 values each)
            float2 v[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) v[t] = sClu[t * NG + tid];
            float c = 2048.f;
#pragma unroll
            for (int w = 8; w > 1; w >>= 1) {
#pragma unroll
                for (int t = 0; t < w / 2; ++t) v[t] = merge2(v[2 * t], v[2 * t + 1], c);
                c *= 2.f;
            }
            const float rstd = rsqrtf(fmaxf(v[0].y * (1.f / 16384.f), 0.f) + a.eps);
            sCoef[64 + tid * 2] = v[0].x;
            sCoef[64 + tid * 2 + 1] = rstd;
        }
        __syncthreads();
        if (tid < C0) {
            const float mean = sCoef[64 + (tid / 16) * 2], rstd = sCoef[64 + (tid / 16) * 2 + 1];
            const float A = rstd * sBN[lgn * 64 + tid];
            sCoef[tid] = A;
            sCoef[32 + tid] = fmaf(-mean, A, sBN[lgn * 64 + 32 + tid]);
        }
        __syncthreads();
    };
    constexpr int NPASS = GN ? 2 : 1;

    for (int img = blockIdx.x / P; img < a.B; img += gridDim.x / P) {
        // ---- the image -> smem (6 KiB, coalesced 16-B loads)
        {
            const uint4 *src = reinterpret_cast<const uint4 *>(a.in + static_cast<size_t>(img) * kFsImg * kFsImg * 3);
            for (int i = tid; i < kFsImgBytes / 16; i += kFsThreads) reinterpret_cast<uint4 *>(pImg)[i] = src[i];
        }
        __syncthreads();
        FS_STAMP();
        // ---- stem: conv3x3 3 -> C0 + norm + ReLU -> X; rounds of up to four tiles (A slots 0..3)
        for (int pass = 2 - NPASS + 1; pass <= 2; ++pass) {
            const float *cA = GN ? sCoef : sBN, *cB = GN ? sCoef + 32 : sBN + 32;
            for (int rnd = 0; rnd * ROUND < TPC; ++rnd) {
                if (warp < kFsEpiWarps && g < ROUND) {   // im2col: one output pixel (A row) per thread
                    const int t = ROUND * rnd + g, h = h_base + 4 * t + q;
                    const uint16_t *im = reinterpret_cast<const uint16_t *>(pImg);
                    uint32_t packed[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) packed[j] = 0;
#pragma unroll
                    for (int kh = 0; kh < 3; ++kh)
#pragma unroll
                        for (int kw = 0; kw < 3; ++kw) {
                            const int ih = h + kh - 1, iw = lane + kw - 1;
                            const bool ok = ih >= 0 && ih < kFsImg && iw >= 0 && iw < kFsImg;
                            const uint16_t *px = im + (ih * kFsImg + iw) * 3;
#pragma unroll
                            for (int ci = 0; ci < 3; ++ci) {
                                const int k = (kh * 3 + kw) * 3 + ci;
                                const uint32_t b = ok ? static_cast<uint32_t>(px[ci]) : 0u;
                                packed[k >> 1] |= (k & 1) ? (b << 16) : b;
                            }
                        }
                    uint8_t *dst = pA + g * 8192;
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        *reinterpret_cast<uint4 *>(dst + swz_off(row, j, 64)) =
                            make_uint4(packed[4 * j], packed[4 * j + 1], packed[4 * j + 2], packed[4 * j + 3]);
                    fence_proxy_async();
                }
                __syncthreads();
                if (warp == kFsEpiWarps) {
                    tc_fence_after();
                    const uint32_t idesc = umma_idesc_bf16(kTileM, C0);
                    const uint64_t bd = umma_desc_kmajor(sWs, 64);
                    for (int gg = 0; gg < ROUND; ++gg) {
                        const uint32_t uu = u + gg, s = uu % S;
                        if (uu >= static_cast<uint32_t>(S)) mbar_wait(t_empty(s), ((uu / S) - 1) & 1);
                        tc_fence_after();
                        if (elect_one()) {
                            const uint64_t ad = umma_desc_kmajor(sA + gg * 8192, 64);
                            umma_bf16(tmem + s * SC, ad, bd, idesc, 0u);
                            umma_bf16(tmem + s * SC, ad + 2, bd + 2, idesc, 1u);
                            umma_commit(t_full(s));
                        }
                        __syncwarp();
                    }
                } else if (g < ROUND) {   // stem epilogue of tile ROUND*rnd + g
                    const int t = ROUND * rnd + g;
                    const uint32_t uu = u + g, s = uu % S;
                    mbar_wait(t_full(s), (uu / S) & 1);
                    tc_fence_after();
#pragma unroll
                    for (int gi = 0; gi < NG; ++gi) {
                        uint32_t v[16];
                        tmem_ld16(lane_addr + s * SC + gi * 16, v);
                        tmem_wait_ld();
                        reg_fence16(v);
                        if (GN && pass == 1) {
                            float y[16];
#pragma unroll
                            for (int i = 0; i < 16; ++i) y[i] = __uint_as_float(v[i]);
                            warp_stats(y, t, gi);
                            continue;
                        }
                        uint32_t o[8];
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const int c = gi * 16 + 2 * i;
                            o[i] = pack_bf16(fmaxf(fmaf(__uint_as_float(v[2 * i]), cA[c], cB[c]), 0.f),
                                             fmaxf(fmaf(__uint_as_float(v[2 * i + 1]), cA[c + 1], cB[c + 1]), 0.f));
                        }
                        store_act(pX, t, 2 * gi, make_uint4(o[0], o[1], o[2], o[3]));
                        store_act(pX, t, 2 * gi + 1, make_uint4(o[4], o[5], o[6], o[7]));
                    }
                    tc_fence_before();
                    mbar_arrive(t_empty(s));
                }
                u += ROUND;
                __syncthreads();   // this round's A slots consumed (each group waited for its MMA) before rebuild
                FS_STAMP();
            }
            if (GN && pass == 1) gn_finish(0);
        }
        layer_sync();
        // ---- the two BasicBlocks: l = 0: X -> T, 1: T -> X (+ X), 2: X -> T, 3: T -> X (+ X) / global
        for (int l = 0; l < 4; ++l) {
            const uint32_t src = (l & 1) ? sT : sX;
            uint8_t *dst = (l & 1) ? pX : pT;
            for (int pass = 2 - NPASS + 1; pass <= 2; ++pass) {
                if (warp == kFsEpiWarps) {
                    const uint32_t idesc = umma_idesc_bf16(kTileM, 3 * C0);
                    for (int t = 0; t < TPC; ++t) {
                        const uint32_t uu = u + t, s = uu % S;
                        if (uu >= static_cast<uint32_t>(S)) mbar_wait(t_empty(s), ((uu / S) - 1) & 1);
                        tc_fence_after();
                        if (elect_one()) {
#pragma unroll
                            for (int kh = 0; kh < 3; ++kh) {
                                const uint64_t ad =
                                    umma_desc_kmajor(src + static_cast<uint32_t>((4 * t + kh) * 32 * RB), RB);
                                const uint64_t bd =
                                    umma_desc_kmajor(sWc + static_cast<uint32_t>((l * 9 + kh * 3) * C0 * RB), RB);
#pragma unroll
                                for (int kk = 0; kk < C0 / 16; ++kk)
                                    umma_bf16(tmem + s * SC, ad + 2 * kk, bd + 2 * kk, idesc, (kh | kk) != 0);
                            }
                            umma_commit(t_full(s));
                        }
                        __syncwarp();
                    }
                } else {
                    const float *sc = GN ? sCoef : sBN + (l + 1) * 64, *sh = sc + 32;
                    const bool res = (l & 1) != 0, last = l == 3;
                    for (int t = g; t < TPC; t += 4) {
                        const uint32_t uu = u + t, s = uu % S;
                        mbar_wait(t_full(s), (uu / S) & 1);
                        tc_fence_after();
                        const uint32_t R = static_cast<uint32_t>((4 * t + q + 1) * 32 + lane);   // local buffer row
                        const int h = h_base + 4 * t + q;
#pragma unroll
                        for (int gi = 0; gi < NG; ++gi) {
                            uint32_t v0[16], v1[16], v2[16];
                            const uint32_t col = lane_addr + s * SC + gi * 16;
                            tmem_ld16(col, v0);
                            tmem_ld16(col + C0, v1);
                            tmem_ld16(col + 2 * C0, v2);
                            tmem_wait_ld();
                            reg_fence16(v0);
                            reg_fence16(v1);
                            reg_fence16(v2);
                            float f[16];
                            const unsigned long long mL2 = f2pk(mL, mL), mR2 = f2pk(mR, mR);
                            if (GN && pass == 1) {   // raw output (acc0[w-1] + acc1[w] + acc2[w+1]) -> statistics
#pragma unroll
                                for (int i = 0; i < 16; i += 2) {
                                    const float l0 = __shfl_up_sync(0xffffffffu, __uint_as_float(v0[i]), 1);
                                    const float l1 = __shfl_up_sync(0xffffffffu, __uint_as_float(v0[i + 1]), 1);
                                    const float r0 = __shfl_down_sync(0xffffffffu, __uint_as_float(v2[i]), 1);
                                    const float r1 = __shfl_down_sync(0xffffffffu, __uint_as_float(v2[i + 1]), 1);
                                    f2upk(ffma2(mR2, f2pk(r0, r1),
                                                ffma2(mL2, f2pk(l0, l1),
                                                      f2pk(__uint_as_float(v1[i]), __uint_as_float(v1[i + 1])))),
                                          f[i], f[i + 1]);
                                }
                                warp_stats(f, t, gi);
                                continue;
                            }
#pragma unroll
                            for (int i = 0; i < 16; i += 2) {   // out[w] = acc0[w-1] + acc1[w] + acc2[w+1], then norm
                                const float l0 = __shfl_up_sync(0xffffffffu, __uint_as_float(v0[i]), 1);
                                const float l1 = __shfl_up_sync(0xffffffffu, __uint_as_float(v0[i + 1]), 1);
                                const float r0 = __shfl_down_sync(0xffffffffu, __uint_as_float(v2[i]), 1);
                                const float r1 = __shfl_down_sync(0xffffffffu, __uint_as_float(v2[i + 1]), 1);
                                const unsigned long long y = ffma2(
                                    mR2, f2pk(r0, r1),
                                    ffma2(mL2, f2pk(l0, l1), f2pk(__uint_as_float(v1[i]), __uint_as_float(v1[i + 1]))));
                                const int c = gi * 16 + i;
                                f2upk(ffma2(y, f2pk(sc[c], sc[c + 1]), f2pk(sh[c], sh[c + 1])), f[i], f[i + 1]);
                            }
                            uint8_t *p0 = dst + swz_off(R, 2 * gi, RB), *p1 = dst + swz_off(R, 2 * gi + 1, RB);
                            if (res) {   // + the block input (in place: this thread's own pixel and channels)
                                const uint4 r0 = *reinterpret_cast<const uint4 *>(p0);
                                const uint4 r1 = *reinterpret_cast<const uint4 *>(p1);
                                const uint32_t rr[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
#pragma unroll
                                for (int i = 0; i < 8; ++i)
                                    f2upk(fadd2(f2pk(f[2 * i], f[2 * i + 1]), f2pk(bf16_lo(rr[i]), bf16_hi(rr[i]))),
                                          f[2 * i], f[2 * i + 1]);
                            }
                            uint32_t o[8];
#pragma unroll
                            for (int i = 0; i < 8; ++i) o[i] = pack_bf16(fmaxf(f[2 * i], 0.f), fmaxf(f[2 * i + 1], 0.f));
                            const uint4 o0 = make_uint4(o[0], o[1], o[2], o[3]), o1 = make_uint4(o[4], o[5], o[6], o[7]);
                            if (last) {   // segment output [B][32][32][C0]
                                uint4 *gp = reinterpret_cast<uint4 *>(
                                    a.out + ((static_cast<size_t>(img) * kFsImg + h) * kFsImg + lane) * C0 + gi * 16);
                                gp[0] = o0;
                                gp[1] = o1;
                            } else {
                                store_act(dst, t, 2 * gi, o0);
                                store_act(dst, t, 2 * gi + 1, o1);
                            }
                        }
                        tc_fence_before();
                        mbar_arrive(t_empty(s));
                    }
                }
                u += TPC;
                if (GN && pass == 1) {
                    tc_fence_before();
                    gn_finish(l + 1);
                    tc_fence_after();
                }
            }
            layer_sync();
            FS_STAMP();
        }
    }
    tc_fence_before();
    if (P > 1)
        cluster_sync_all();
    else
        __syncthreads();
    if (warp == kFsEpiWarps) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
    }
}

}  // namespace

size_t seg0_fused_smem_bytes(int c0, int P) { return 1024 + fs_layout(c0, P).total; }

cudaError_t launch_seg0_fused(const FusedSeg0Args &a, int grid, cudaStream_t stream, bool pdl) {
    if (a.c0 != 16 && a.c0 != 32) return cudaErrorInvalidValue;
    const int P = a.cluster == 8 ? 8 : 1;
    using Fn = void (*)(FusedSeg0Args);
    const Fn fns[2][2][2] = {{{seg0_fused_kernel<16, 1, false>, seg0_fused_kernel<16, 1, true>},
                              {seg0_fused_kernel<16, 8, false>, seg0_fused_kernel<16, 8, true>}},
                             {{seg0_fused_kernel<32, 1, false>, seg0_fused_kernel<32, 1, true>},
                              {seg0_fused_kernel<32, 8, false>, seg0_fused_kernel<32, 8, true>}}};
    const Fn fn = fns[a.c0 == 32][P == 8][a.gn ? 1 : 0];
    const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(seg0_fused_smem_bytes(a.c0, P)));
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid * P);
    cfg.blockDim = dim3(kFsThreads);
    cfg.dynamicSmemBytes = seg0_fused_smem_bytes(a.c0, P);
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = P;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, fn, a);
}

namespace {

// =====================================================================================================
// Segments 1-3 as ONE kernel for the narrow widths: block 0 (3x3 stride-2 conv + BN + ReLU; 3x3 conv +
// BN + 1x1 stride-2 projection + BN + ReLU) and block 1 (two 3x3 convs, identity shortcut), segment 3
// ending in the fused global average pool.  A cluster of P CTAs takes a UNIT of G images (G*H*W = 128
// or 256 output pixels: segment 1 H=16 G=1, segment 2 H=8 G=2, segment 3 H=4 G=8) through all four
// layers with every activation in shared memory; CTA p of the cluster computes output channels
// [p*R, (p+1)*R), R = C/P, and writes them into the activation buffers of every CTA of the cluster
// (DSMEM), so each CTA holds the whole layer output as the next layer's A operand; a layer boundary is
// a local barrier plus one remote mbarrier arrive per peer.  Weights stream through a ring of slabs (one
// 1-D bulk copy each, from a pre-swizzled per-rank image built at load, build_segn_fused_image) in
// exactly the order the MMAs use them.  Bit-identical to the per-layer halo kernels: the same MMAs in
// the same K order (stride 2: kh 0, 2, 1 with [kw0 | kw2] on the odd-column plane and kw1 on the even
// one; stride 1: chunk outer, kh, 16-channel steps; an output column's sum does not depend on how the
// N dimension is split), the same epilogue arithmetic.
//
// Activation layout: a "halo row" = RP = G*W pixels ordered (image n, column w); a buffer holds H+2
// halo rows (zero rows 0 and H+1), channels in chunks of <= 64 (K-major, swizzle span = 2*chunk B).
// Stride-2 input: four parity planes of the previous segment's output (row parity x column parity):
// odd-row planes have a zero row 0 (input row -1), index (y+1)/2; even-row planes index y/2; odd-column
// index (x-1)/2, even-column x/2 (the kw=0 tap's w-1 shift is the epilogue's shfl_up, as in the halo
// kernel).  The 1x1 projection reads the even/even plane.
// =====================================================================================================

constexpr int kFnEpiWarps = 16;
constexpr int kFnThreads = (kFnEpiWarps + 2) * 32;   // warps 0-15 epilogue / loaders, 16 MMA, 17 weight producer

__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster_v4(uint32_t addr, uint4 v) {
    asm volatile("st.shared::cluster.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t remote_bar) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_bar) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
}
__device__ __forceinline__ void fence_proxy_async_cluster() {
    asm volatile("fence.proxy.async.shared::cluster;" ::: "memory");
}

struct FnGeom {
    uint32_t rb_i, nch_i, rb_c, nch_c, rp;
    uint32_t plane_odd, plane_even;       // one parity plane (all input chunks)
    uint32_t act;                         // T or X (all C channels)
    uint32_t slot, n_slots;
    uint32_t planes, t, x, ring, bn, bars, gn, total;
};
__host__ __device__ inline uint32_t fn_al(uint32_t v) { return (v + 1023u) & ~1023u; }
__host__ __device__ inline int fn_ck(int c) { return c <= 16 ? 16 : (c <= 32 ? 32 : 64); }
// smem layout for full width C, R = C/P rows per CTA, input width CI; the weight ring takes what the
// budget leaves (up to 6 slots)
__host__ __device__ inline FnGeom fn_layout(int C, int R, int CI, int H, int G, uint32_t budget, bool gn = false) {
    FnGeom g;
    g.rb_i = 2u * fn_ck(CI);
    g.nch_i = (CI + 63) / 64;
    g.rb_c = 2u * fn_ck(C);
    g.nch_c = (C + 63) / 64;
    g.rp = static_cast<uint32_t>(G * H);                          // W == H
    g.plane_odd = fn_al(g.nch_i * (H + 1) * g.rp * g.rb_i);
    g.plane_even = fn_al(g.nch_i * H * g.rp * g.rb_i);
    g.act = fn_al(g.nch_c * (H + 2) * g.rp * g.rb_c);
    const uint32_t taps = 3 * R > 256 ? 1u : 3u;
    g.slot = fn_al(taps * R * (g.rb_i > g.rb_c ? g.rb_i : g.rb_c));
    g.planes = 0;
    g.t = g.planes + 2 * g.plane_odd + 2 * g.plane_even;
    g.x = g.t + g.act;
    g.ring = g.x + g.act;
    const uint32_t gnb = gn ? 6144u : 0u;                      // GroupNorm partials + per-image coefficients
    const uint32_t tail = 5u * 2u * C * 4u + 64u * 8u + 16u + gnb;   // BN / GN vectors, barriers, tmem slot
    uint32_t ns = 0;
    while (ns < 6 && g.ring + (ns + 1) * g.slot + tail <= budget) ++ns;
    g.n_slots = ns;
    g.bn = g.ring + ns * g.slot;
    g.bars = g.bn + 5u * 2u * C * 4u;
    g.gn = g.bars + 64u * 8u + 16u;
    g.total = g.gn + gnb;
    return g;
}

template <int C, int H, int G, int P, bool GN>
__global__ void __launch_bounds__(kFnThreads, 1) segn_fused_kernel(const FusedSegArgs a) {
    constexpr int W = H, RP = G * W, NPIX = G * H * W, NT = NPIX / 128, TR = 128 / RP;
    constexpr int R = C / P;                                 // output channels of this CTA
    constexpr bool TAPM = 3 * R > 256;                       // one tap per slab / MMA
    constexpr int NG = R / 16;                               // 16-channel groups of this CTA
    constexpr int SC = 4 * R;                                // TMEM columns per tile stage: 3 kw accs + projection
    static_assert(NT * SC <= 512, "TMEM");
    const int CI = a.CI;
    const FnGeom Gm = fn_layout(C, R, CI, H, G, a.smem_budget, GN);
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t s0 = smem_u32(smem);
    const uint32_t sPl = s0 + Gm.planes, sT = s0 + Gm.t, sX = s0 + Gm.x, sRing = s0 + Gm.ring;
    // plane (py, px): even-row planes first (px = 0, 1), then odd-row planes
    auto plane_base = [&](int py, int px) -> uint32_t {
        return (py ? 2 * Gm.plane_even + px * Gm.plane_odd : px * Gm.plane_even);
    };
    float *sBN = reinterpret_cast<float *>(smem + Gm.bn);   // [layer][scale C | shift C]
    const uint32_t bar0 = s0 + Gm.bars;
    auto w_full = [&](int i) { return bar0 + 8u * i; };
    auto w_empty = [&](int i) { return bar0 + 8u * (8 + i); };
    auto t_full = [&](int t) { return bar0 + 8u * (16 + t); };
    const uint32_t peer_done = bar0 + 8u * 24;               // P-1 remote arrivals per layer
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + Gm.bars + 64 * 8);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rbi = Gm.rb_i, rbc = Gm.rb_c, nchi = Gm.nch_i;
    const int n_units = (a.B + G - 1) / G;
    const uint32_t rank = P > 1 ? cluster_ctarank() : 0;
    const int unit0 = blockIdx.x / P, unit_step = gridDim.x / P;
    // diagnostics: CTA 0, thread 0 (epilogue) stamps [0..15], the MMA warp's lane 0 [16..31], producer [32..47]
    unsigned long long *tr = (a.trace && blockIdx.x == 0) ? a.trace : nullptr;
    int ntr = 0, ntm = 16, ntp = 32;
#define FN_STAMP()                                                                      \
    do {                                                                                \
        if (tr && tid == 0 && ntr < 16) tr[ntr++] = gtimer();                           \
        if (tr && warp == kFnEpiWarps && lane == 0 && ntm < 32) tr[ntm++] = gtimer();   \
        if (tr && warp == kFnEpiWarps + 1 && lane == 0 && ntp < 48) tr[ntp++] = gtimer(); \
    } while (0)
    FN_STAMP();

    // ---- prologue (static data only: before the PDL wait)
    for (int i = tid; i < 5 * C; i += kFnThreads) {
        const int l = i / C, c = i % C;
        sBN[l * 2 * C + c] = a.scale[l][c];
        sBN[l * 2 * C + C + c] = a.shift[l][c];
    }
    // zero rows: odd-row planes' row 0, T and X rows 0 and H+1 (never written afterwards)
    for (int px = 0; px < 2; ++px) {
        const uint32_t base = Gm.planes + plane_base(1, px);
        for (uint32_t ch = 0; ch < nchi; ++ch)
            for (int i = tid; i < RP * static_cast<int>(rbi) / 16; i += kFnThreads)
                reinterpret_cast<uint4 *>(smem + base + ch * (H + 1) * RP * rbi)[i] = make_uint4(0, 0, 0, 0);
    }
    for (int b = 0; b < 2; ++b)
        for (uint32_t ch = 0; ch < Gm.nch_c; ++ch)
            for (int r = 0; r < 2; ++r)
                for (int i = tid; i < RP * static_cast<int>(rbc) / 16; i += kFnThreads)
                    reinterpret_cast<uint4 *>(smem + (b ? Gm.x : Gm.t) + ch * (H + 2) * RP * rbc +
                                              (r ? (H + 1) * RP * rbc : 0))[i] = make_uint4(0, 0, 0, 0);
    if (tid == 0) {
        for (int i = 0; i < 8; ++i) {
            mbar_init(w_full(i), 1);
            mbar_init(w_empty(i), 1);
            mbar_init(t_full(i), 1);
        }
        mbar_init(peer_done, P > 1 ? P - 1 : 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kFnEpiWarps) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    fence_proxy_async();
    tc_fence_before();
    if (P > 1)
        cluster_sync_all();   // every CTA's barriers are initialised before any remote arrive / store
    else
        __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    FN_STAMP();

    // slab sequence of one unit (identical for producer and MMA issuer): L1: (ch_i, kh in 0,2,1) x
    // [3 taps | tap]; L2: (ch_c, kh) x taps, then the projection (ch_i); L3, L4: (ch_c, kh) x taps
    const int tps = TAPM ? 3 : 1;                            // slabs per (chunk, kh)
    const int n_l1 = nchi * 3 * tps, n_l2 = Gm.nch_c * 3 * tps, n_p = nchi;
    const int n_slabs = n_l1 + n_l2 + n_p + 2 * n_l2;
    auto slab_bytes = [&](int k) -> uint32_t {
        const uint32_t taps = TAPM ? 1u : 3u;
        if (k < n_l1) return taps * R * rbi;
        k -= n_l1;
        if (k < n_l2) return taps * R * rbc;
        k -= n_l2;
        if (k < n_p) return static_cast<uint32_t>(R) * rbi;
        return taps * R * rbc;
    };

    if (warp == kFnEpiWarps + 1) {
        // ===================== weight producer: this rank's slabs in consumption order, every unit ======
        pdl_launch_dependents();
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int u = unit0; u < n_units; u += unit_step) {
                const uint8_t *src = a.wimg + static_cast<size_t>(rank) * a.wimg_rank_bytes;
                for (int k = 0; k < n_slabs; ++k) {
                    const uint32_t by = slab_bytes(k);
                    mbar_wait(w_empty(s), ph ^ 1);
                    mbar_expect_tx(w_full(s), by);
                    bulk_load_1d(sRing + s * Gm.slot, src, by, w_full(s));
                    src += by;
                    if (++s == static_cast<int>(Gm.n_slots)) {
                        s = 0;
                        ph ^= 1;
                    }
                    if ((k & 3) == 3) FN_STAMP();
                }
            }
        }
    } else {
        pdl_wait();
        pdl_launch_dependents();
        FN_STAMP();

        const int q = warp & 3, sub = warp >> 2;             // epilogue: TMEM lane quarter, column way
        const int m = q * 32 + lane;                         // row within a tile
        const int wcol = m % W;                              // pixel column (W divides 32)
        const float mL = wcol > 0 ? 1.f : 0.f, mR = wcol < W - 1 ? 1.f : 0.f;
        const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
        int ws = 0;                                          // MMA: weight ring position
        uint32_t wph = 0;
        uint32_t layers_done = 0;                            // layers completed by this CTA (t_full / peer phases)
        constexpr uint32_t kBarThreads = (kFnEpiWarps + 1) * 32;

        for (int u = unit0; u < n_units; u += unit_step) {
            // ---- the unit's input -> four parity planes (16-B pieces; images past B are zeros)
            if (warp < kFnEpiWarps) {
                const int per_px = CI / 8;                   // 16-B pieces per input pixel
                const int total = G * (2 * H) * (2 * W) * per_px;
                constexpr int kU = 8;                        // loads in flight per thread before the stores
                for (int i0 = tid; i0 < total; i0 += kU * kFnEpiWarps * 32) {
                    uint4 v[kU];
#pragma unroll
                    for (int k = 0; k < kU; ++k) {
                        const int i = i0 + k * kFnEpiWarps * 32;
                        const int j = i % per_px, p = i / per_px;
                        const int img = u * G + p / (4 * H * W);
                        v[k] = make_uint4(0, 0, 0, 0);
                        if (i < total && img < a.B)
                            v[k] = *reinterpret_cast<const uint4 *>(a.in + (static_cast<size_t>(u * G) * 4 * H * W + p) * CI +
                                                                    j * 8);
                    }
#pragma unroll
                    for (int k = 0; k < kU; ++k) {
                        const int i = i0 + k * kFnEpiWarps * 32;
                        if (i >= total) break;
                        const int j = i % per_px, p = i / per_px;
                        const int x = p % (2 * W), y = (p / (2 * W)) % (2 * H), n = p / (4 * H * W);
                        const int py = y & 1, px = x & 1;
                        const int row = py ? (y + 1) / 2 : y / 2, col = px ? (x - 1) / 2 : x / 2;
                        const int ch = (j * 8) / 64, jj = j % (static_cast<int>(rbi) / 16);
                        const uint32_t rows = py ? (H + 1) : H;
                        const uint32_t off = Gm.planes + plane_base(py, px) + ch * rows * RP * rbi +
                                             swz_off(row * RP + n * W + col, jj, rbi);
                        *reinterpret_cast<uint4 *>(smem + off) = v[k];
                    }
                }
                fence_proxy_async();
            }
            named_bar_sync(1, kBarThreads);
            tc_fence_after();
            FN_STAMP();
            for (int l = 1; l <= 4; ++l) {
                if (warp == kFnEpiWarps) {
                    // ===================== MMA issuer ====================================================
                    // the previous layer's outputs of every peer are in this CTA's buffers (and the peers
                    // are done reading the buffer this layer's epilogue will write into theirs)
                    if (P > 1 && layers_done > 0) mbar_wait_cluster(peer_done, (layers_done - 1) & 1);
                    tc_fence_after();
                    const uint32_t src = (l == 2 || l == 4) ? sT : sX;   // L2, L4 read T; L3 reads X
                    auto next_slab = [&]() -> uint32_t {
                        mbar_wait(w_full(ws), wph);
                        tc_fence_after();
                        return sRing + ws * Gm.slot;
                    };
                    auto release_slab = [&]() {
                        if (elect_one()) umma_commit(w_empty(ws));
                        __syncwarp();
                        if (++ws == static_cast<int>(Gm.n_slots)) {
                            ws = 0;
                            wph ^= 1;
                        }
                    };
                    if (l == 1) {
                        // stride-2 conv from the parity planes: kh order 0, 2, 1
                        const uint32_t idesc1 = umma_idesc_bf16(kTileM, R), idesc2 = umma_idesc_bf16(kTileM, 2 * R);
                        for (uint32_t ch = 0; ch < nchi; ++ch) {
                            const int nk = min(static_cast<int>(rbi) / 32, (CI - static_cast<int>(ch) * 64 + 15) >> 4);
                            for (int o = 0; o < 3; ++o) {
                                const int kh = o == 0 ? 0 : (o == 1 ? 2 : 1);
                                const int py = kh == 1 ? 0 : 1, roff = kh == 2 ? 1 : 0;
                                const uint32_t rows = py ? (H + 1) : H;
                                for (int j = 0; j < (TAPM ? 3 : 1); ++j) {
                                    const uint32_t sb = next_slab();
                                    if (elect_one()) {
                                        for (int t = 0; t < NT; ++t) {
                                            const uint32_t acc = tmem + t * SC;
                                            const uint32_t aoff = ch * rows * RP * rbi + (t * TR + roff) * RP * rbi;
                                            const uint64_t aod = umma_desc_kmajor(sPl + plane_base(py, 1) + aoff, rbi);
                                            const uint64_t aev = umma_desc_kmajor(sPl + plane_base(py, 0) + aoff, rbi);
                                            const uint64_t bd = umma_desc_kmajor(sb, rbi);
                                            for (int kk = 0; kk < nk; ++kk) {
                                                const uint32_t accum = (ch | kh | kk) != 0;
                                                if (!TAPM) {   // slab taps [kw0 | kw2 | kw1]
                                                    umma_bf16(acc, aod + 2 * kk, bd + 2 * kk, idesc2, accum);
                                                    umma_bf16(acc + 2 * R, aev + 2 * kk,
                                                              bd + ((2u * R * rbi) >> 4) + 2 * kk, idesc1, accum);
                                                } else if (j < 2) {   // tap kw0 -> acc0, kw2 -> acc1 (odd columns)
                                                    umma_bf16(acc + j * R, aod + 2 * kk, bd + 2 * kk, idesc1, accum);
                                                } else {              // kw1 -> acc2 (even columns)
                                                    umma_bf16(acc + 2 * R, aev + 2 * kk, bd + 2 * kk, idesc1, accum);
                                                }
                                            }
                                        }
                                    }
                                    __syncwarp();
                                    release_slab();
                                }
                            }
                        }
                    } else {
                        const uint32_t idesc3 = umma_idesc_bf16(kTileM, TAPM ? R : 3 * R),
                                       idesc1 = umma_idesc_bf16(kTileM, R);
                        for (uint32_t ch = 0; ch < Gm.nch_c; ++ch) {
                            const int nk = min(static_cast<int>(rbc) / 32, (C - static_cast<int>(ch) * 64 + 15) >> 4);
                            for (int kh = 0; kh < 3; ++kh) {
                                for (int j = 0; j < (TAPM ? 3 : 1); ++j) {
                                    const uint32_t sb = next_slab();
                                    if (elect_one()) {
                                        for (int t = 0; t < NT; ++t) {
                                            const uint32_t acc = tmem + t * SC + (TAPM ? j * R : 0);
                                            const uint64_t ad = umma_desc_kmajor(
                                                src + ch * (H + 2) * RP * rbc + (t * TR + kh) * RP * rbc, rbc);
                                            const uint64_t bd = umma_desc_kmajor(sb, rbc);
                                            for (int kk = 0; kk < nk; ++kk)
                                                umma_bf16(acc, ad + 2 * kk, bd + 2 * kk, idesc3, (ch | kh | kk) != 0);
                                        }
                                    }
                                    __syncwarp();
                                    release_slab();
                                }
                            }
                        }
                        if (l == 2) {   // 1x1 stride-2 projection from the even/even plane -> 4th accumulator
                            for (uint32_t cp = 0; cp < nchi; ++cp) {
                                const int nk =
                                    min(static_cast<int>(rbi) / 32, (CI - static_cast<int>(cp) * 64 + 15) >> 4);
                                const uint32_t sb = next_slab();
                                if (elect_one()) {
                                    for (int t = 0; t < NT; ++t) {
                                        const uint64_t ad = umma_desc_kmajor(
                                            sPl + plane_base(0, 0) + cp * H * RP * rbi + t * TR * RP * rbi, rbi);
                                        const uint64_t bd = umma_desc_kmajor(sb, rbi);
                                        for (int kk = 0; kk < nk; ++kk)
                                            umma_bf16(tmem + t * SC + 3 * R, ad + 2 * kk, bd + 2 * kk, idesc1,
                                                      (cp | kk) != 0);
                                    }
                                }
                                __syncwarp();
                                release_slab();
                            }
                        }
                    }
                    if (elect_one())
                        for (int t = 0; t < NT; ++t) umma_commit(t_full(t));
                    __syncwarp();
                    FN_STAMP();
                } else {
                    // ===================== epilogue: items (tile, 16-channel group) over the 4 column ways ==
                    const int bn_l = l == 1 ? 0 : (l == 2 ? 1 : l);   // BN slots: b0c1, b0c2, sc, b1c1, b1c2
                    const float *sc = sBN + bn_l * 2 * C, *sh = sc + C;
                    const float *sc1 = sBN + 2 * 2 * C, *sh1 = sc1 + C;
                    const uint32_t dstb = (l == 2) ? Gm.x : Gm.t;     // L1, L3 -> T; L2 -> X; L4 -> global
                    const bool pool = a.pool_out != nullptr && l == 4;
                    // L4 pool partials: the even-row planes (dead after L2's projection; no zero rows to keep)
                    float *stage = reinterpret_cast<float *>(smem + Gm.planes);
                    // GroupNorm: pass 1 the statistics per (image of the unit, 16-channel group) of the fp32 raw
                    // outputs (u; and the projection p at L2) -- per thread (mean, M2) of 16 values, merged with
                    // equal counts over the lanes of the same image, then over (tile, lane quarter) in a fixed
                    // tree -- pass 2 the normalisation with per-(image, channel) coefficients.  The accumulators
                    // stay in TMEM between the passes (a unit's tiles never share a stage).
                    constexpr int SLOTS = RP / W;                                   // images per warp row
                    const float leaf_cnt = 16.f * 32.f * W / RP;
                    float2 *gPart = reinterpret_cast<float2 *>(smem + Gm.gn);      // [which][t][q][gi][slot]
                    float *gCoef = reinterpret_cast<float *>(gPart + 2 * NT * 4 * NG * SLOTS);   // [which][A|B][n][cl]
                    auto gpart = [&](int which, int t, int qq, int gi_, int slot) -> float2 & {
                        return gPart[(((which * NT + t) * 4 + qq) * NG + gi_) * SLOTS + slot];
                    };
                    auto stats16 = [&](const float (&y)[16], int which, int t, int gi_) {
                        float mu = 0.f;
#pragma unroll
                        for (int i = 0; i < 16; ++i) mu += y[i];
                        mu *= (1.f / 16.f);
                        float m2 = 0.f;
#pragma unroll
                        for (int i = 0; i < 16; ++i) m2 = fmaf(y[i] - mu, y[i] - mu, m2);
                        float cnt = 16.f;
                        for (int ofs = 1; ofs < 32; ofs <<= 1) {
                            if (ofs >= W && ofs < RP) continue;   // would mix images
                            const float mo = __shfl_xor_sync(0xffffffffu, mu, ofs), qo = __shfl_xor_sync(0xffffffffu, m2, ofs);
                            const float d = mo - mu;
                            m2 = (m2 + qo) + d * d * (cnt * 0.5f);
                            mu = (mu + mo) * 0.5f;
                            cnt *= 2.f;
                        }
                        if (lane < RP && lane % W == 0) gpart(which, t, q, gi_, lane / W) = make_float2(mu, m2);
                    };
                    for (int pass = GN ? 1 : 2; pass <= 2; ++pass) {
                    if (GN && pass == 2) {   // pass-1 partials -> per (image, channel) coefficients
                        named_bar_sync(2, kFnEpiWarps * 32);
                        const int nwhich = l == 2 ? 2 : 1;
                        for (int idx = tid; idx < nwhich * G * NG; idx += kFnEpiWarps * 32) {
                            const int which = idx / (G * NG), n = (idx / NG) % G, gi_ = idx % NG;
                            float2 lv[2 * NT];
                            float c = leaf_cnt;
#pragma unroll
                            for (int t = 0; t < NT; ++t) {   // quarters pairwise, then the tiles
                                const float2 a0 = gpart(which, t, 0, gi_, n), a1 = gpart(which, t, 1, gi_, n);
                                const float2 a2 = gpart(which, t, 2, gi_, n), a3 = gpart(which, t, 3, gi_, n);
                                auto mg = [](float2 x, float2 y, float cc) {
                                    const float d = y.x - x.x;
                                    return make_float2((x.x + y.x) * 0.5f, (x.y + y.y) + d * d * (cc * 0.5f));
                                };
                                lv[t] = mg(mg(a0, a1, c), mg(a2, a3, c), 2.f * c);
                            }
                            float2 tot = lv[0];
                            float cc = 4.f * c;
                            for (int t = 1; t < NT; ++t) {   // NT <= 2
                                const float d = lv[t].x - tot.x;
                                tot = make_float2((tot.x + lv[t].x) * 0.5f, (tot.y + lv[t].y) + d * d * (cc * 0.5f));
                                cc *= 2.f;
                            }
                            const float rstd = rsqrtf(fmaxf(tot.y / cc, 0.f) + a.eps);
                            const int bl = which ? 2 : bn_l;   // gamma / beta slots (projection: slot 2)
                            for (int i = 0; i < 16; ++i) {
                                const int cl = gi_ * 16 + i, cgl = static_cast<int>(rank) * R + cl;
                                const float A = rstd * sBN[bl * 2 * C + cgl];
                                gCoef[((which * 2 + 0) * G + n) * R + cl] = A;
                                gCoef[((which * 2 + 1) * G + n) * R + cl] = fmaf(-tot.x, A, sBN[bl * 2 * C + C + cgl]);
                            }
                        }
                        named_bar_sync(2, kFnEpiWarps * 32);
                    }
                    for (int it = sub; it < NT * NG; it += 4) {
                        const int t = it / NG, gi = it % NG;
                        // (GN pass 2 reads the accumulators pass 1 already waited for)
                        if (!GN || pass == 1) mbar_wait(t_full(t), layers_done & 1);
                        tc_fence_after();
                        const int hr = t * TR + m / RP, pix = m % RP, n = pix / W;   // output row, image in unit
                        const int cg = static_cast<int>(rank) * R + gi * 16;         // first global channel
                        uint32_t v0[16], v1[16], v2[16];
                        const uint32_t col = tmem + lane_off + t * SC + gi * 16;
                        tmem_ld16(col, v0);
                        tmem_ld16(col + R, v1);
                        tmem_ld16(col + 2 * R, v2);
                        tmem_wait_ld();
                        reg_fence16(v0);
                        reg_fence16(v1);
                        reg_fence16(v2);
                        float f[16];
                        // normalisation coefficients: BN per channel, or GN per (image, channel) (pass 2)
                        const float *ca = GN ? gCoef + (0 * G + n) * R + gi * 16 - cg : sc;
                        const float *cb = GN ? gCoef + (1 * G + n) * R + gi * 16 - cg : sh;
                        if (GN && pass == 1) {   // raw outputs -> statistics
                            if (l == 1) {
#pragma unroll
                                for (int i = 0; i < 16; ++i) {
                                    const float left = __shfl_up_sync(0xffffffffu, __uint_as_float(v0[i]), 1);
                                    f[i] = fmaf(mL, left, __uint_as_float(v1[i]) + __uint_as_float(v2[i]));
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
                                                ffma2(mL2, f2pk(l0, l1),
                                                      f2pk(__uint_as_float(v1[i]), __uint_as_float(v1[i + 1])))),
                                          f[i], f[i + 1]);
                                }
                            }
                            stats16(f, 0, t, gi);
                            if (l == 2) {   // the projection's raw output
                                tmem_ld16(col + 3 * R, v0);
                                tmem_wait_ld();
                                reg_fence16(v0);
#pragma unroll
                                for (int i = 0; i < 16; ++i) f[i] = __uint_as_float(v0[i]);
                                stats16(f, 1, t, gi);
                            }
                            continue;
                        }
                        if (l == 1) {   // acc [kw0 | kw2 | kw1]: kw0[w-1] + kw2[w] + kw1[w] (scalar, as the halo kernel)
#pragma unroll
                            for (int i = 0; i < 16; ++i) {
                                const float left = __shfl_up_sync(0xffffffffu, __uint_as_float(v0[i]), 1);
                                const float y = fmaf(mL, left, __uint_as_float(v1[i]) + __uint_as_float(v2[i]));
                                f[i] = fmaf(y, ca[cg + i], cb[cg + i]);
                            }
                        } else {
                            const unsigned long long mL2 = f2pk(mL, mL), mR2 = f2pk(mR, mR);
#pragma unroll
                            for (int i = 0; i < 16; i += 2) {
                                const float l0 = __shfl_up_sync(0xffffffffu, __uint_as_float(v0[i]), 1);
                                const float l1 = __shfl_up_sync(0xffffffffu, __uint_as_float(v0[i + 1]), 1);
                                const float r0 = __shfl_down_sync(0xffffffffu, __uint_as_float(v2[i]), 1);
                                const float r1 = __shfl_down_sync(0xffffffffu, __uint_as_float(v2[i + 1]), 1);
                                const unsigned long long y = ffma2(
                                    mR2, f2pk(r0, r1),
                                    ffma2(mL2, f2pk(l0, l1), f2pk(__uint_as_float(v1[i]), __uint_as_float(v1[i + 1]))));
                                const int c = cg + i;
                                f2upk(ffma2(y, f2pk(ca[c], ca[c + 1]), f2pk(cb[c], cb[c + 1])), f[i], f[i + 1]);
                            }
                        }
                        if (l == 2) {   // + s_sc * proj + t_sc (GN: the projection's own GN)
                            const float *pa = GN ? gCoef + (2 * G + n) * R + gi * 16 - cg : sc1;
                            const float *pb = GN ? gCoef + (3 * G + n) * R + gi * 16 - cg : sh1;
                            tmem_ld16(col + 3 * R, v0);
                            tmem_wait_ld();
                            reg_fence16(v0);
#pragma unroll
                            for (int i = 0; i < 16; i += 2) {
                                const int c = cg + i;
                                const unsigned long long pr =
                                    ffma2(f2pk(__uint_as_float(v0[i]), __uint_as_float(v0[i + 1])),
                                          f2pk(pa[c], pa[c + 1]), f2pk(pb[c], pb[c + 1]));
                                f2upk(fadd2(f2pk(f[i], f[i + 1]), pr), f[i], f[i + 1]);
                            }
                        }
                        // this pixel in the activation buffers: halo row hr+1, chunk cg/64
                        const uint32_t chk = cg / 64, pc = (cg % 64) / 8;
                        const uint32_t brow = (hr + 1) * RP + pix;
                        const uint32_t o0 = chk * (H + 2) * RP * rbc + swz_off(brow, pc, rbc);
                        const uint32_t o1 = chk * (H + 2) * RP * rbc + swz_off(brow, pc + 1, rbc);
                        if (l == 4) {   // + the block input (X, this pixel)
                            const uint4 r0 = *reinterpret_cast<const uint4 *>(smem + Gm.x + o0);
                            const uint4 r1 = *reinterpret_cast<const uint4 *>(smem + Gm.x + o1);
                            const uint32_t rr[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
#pragma unroll
                            for (int i = 0; i < 8; ++i)
                                f2upk(fadd2(f2pk(f[2 * i], f[2 * i + 1]), f2pk(bf16_lo(rr[i]), bf16_hi(rr[i]))),
                                      f[2 * i], f[2 * i + 1]);
                        }
                        if (pool) {
                            // fused global average pool, as the halo kernel: the W pixels of an image row summed
                            // across lanes, parked per (row, image, channel); rows summed below in fixed order
#pragma unroll
                            for (int i = 0; i < 16; ++i) f[i] = fmaxf(f[i], 0.f);
                            for (int o = 1; o < W; o <<= 1) {
#pragma unroll
                                for (int i = 0; i < 16; ++i) f[i] += __shfl_xor_sync(0xffffffffu, f[i], o);
                            }
                            if (wcol == 0) {
                                float4 *dstp = reinterpret_cast<float4 *>(stage + (hr * G + n) * R + gi * 16);
#pragma unroll
                                for (int i = 0; i < 4; ++i)
                                    dstp[i] = make_float4(f[4 * i], f[4 * i + 1], f[4 * i + 2], f[4 * i + 3]);
                            }
                            continue;
                        }
                        uint32_t o[8];
#pragma unroll
                        for (int i = 0; i < 8; ++i) o[i] = pack_bf16(fmaxf(f[2 * i], 0.f), fmaxf(f[2 * i + 1], 0.f));
                        const uint4 q0 = make_uint4(o[0], o[1], o[2], o[3]), q1 = make_uint4(o[4], o[5], o[6], o[7]);
                        if (l == 4) {
                            const int img = u * G + n;
                            if (img < a.B) {
                                uint4 *gp = reinterpret_cast<uint4 *>(
                                    a.out + ((static_cast<size_t>(img) * H + hr) * W + wcol) * C + cg);
                                gp[0] = q0;
                                gp[1] = q1;
                            }
                        } else {
                            *reinterpret_cast<uint4 *>(smem + dstb + o0) = q0;
                            *reinterpret_cast<uint4 *>(smem + dstb + o1) = q1;
#pragma unroll
                            for (int pr = 1; pr < P; ++pr) {   // the same slice into every peer's buffer
                                const uint32_t peer = (rank + pr) % P;
                                st_cluster_v4(mapa_shared(s0 + dstb + o0, peer), q0);
                                st_cluster_v4(mapa_shared(s0 + dstb + o1, peer), q1);
                            }
                        }
                    }
                    }   // passes
                    if (P > 1)
                        fence_proxy_async_cluster();
                    else
                        fence_proxy_async();
                    tc_fence_before();
                    if (pool) {   // rows summed in order h = 0..H-1, times 1/(H*W)
                        named_bar_sync(2, kFnEpiWarps * 32);
                        const float inv = 1.f / static_cast<float>(H * W);
                        for (int idx = tid; idx < G * R; idx += kFnEpiWarps * 32) {
                            float sum = 0.f;
                            for (int h = 0; h < H; ++h) sum += stage[h * G * R + idx];
                            const int img = u * G + idx / R;
                            if (img < a.B)
                                a.pool_out[static_cast<size_t>(img) * C + rank * R + idx % R] = sum * inv;
                        }
                    }
                }
                ++layers_done;
                if (warp < kFnEpiWarps) FN_STAMP();
                named_bar_sync(1, kBarThreads);
                tc_fence_after();
                if (P > 1 && tid == 0) {   // this CTA's slice of the layer is in every peer's buffers
#pragma unroll
                    for (int pr = 1; pr < P; ++pr) mbar_arrive_remote(mapa_shared(peer_done, (rank + pr) % P));
                }
            }
        }
    }
    tc_fence_before();
    if (P > 1)
        cluster_sync_all();   // no CTA exits while a peer may still write into it or arrive on its barrier
    else
        __syncthreads();
    if (warp == kFnEpiWarps) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
    }
}

int fn_geom_seg(int seg, int *H, int *G) {
    *H = 32 >> seg;
    *G = seg == 1 ? 1 : (seg == 2 ? 2 : 8);
    return 0;
}

}  // namespace

// cluster size of the fused segment kernel for (seg, C): output channels split over P CTAs where a single
// CTA would be weight-streaming / MMA bound (8-image segment-3 units; segment 2 at C = 128)
int segn_fused_cluster(int seg, int C) {
    if (seg == 3) return C >= 128 ? 4 : 2;
    if (seg == 2 && C >= 128) return 2;
    return 1;
}

// smem the fused segment-s kernel needs for (C, CI) at segment s (0 if unsupported); >= 2 ring slots
size_t segn_fused_smem_bytes(int seg, int C, int CI, bool gn) {
    if (!(seg >= 1 && seg <= 3) || (C != 32 && C != 64 && C != 128) || CI % 16 != 0 || CI > 128) return 0;
    if (seg == 1 && C == 128) return 0;
    int H, G;
    fn_geom_seg(seg, &H, &G);
    const int P = segn_fused_cluster(seg, C), R = C / P;
    if (G * H * H / 128 * 4 * R > 512) return 0;
    const FnGeom g = fn_layout(C, R, CI, H, G, 227u * 1024u - 1024u, gn);
    if (g.n_slots < 2) return 0;
    return 1024 + g.total;
}

// bytes of one rank's weight image (R = C/P output rows) for (C, CI): slabs in consumption order
size_t segn_fused_rank_image_bytes(int seg, int C, int CI) {
    const int R = C / segn_fused_cluster(seg, C);
    const int ck_i = fn_ck(CI), ck_c = fn_ck(C);
    const size_t nchi = (CI + 63) / 64, nchc = (C + 63) / 64;
    return static_cast<size_t>(R) * (9 * nchi * 2 * ck_i + 3 * 9 * nchc * 2 * ck_c + nchi * 2 * ck_i);
}
size_t segn_fused_image_bytes(int seg, int C, int CI) {
    return segn_fused_cluster(seg, C) * segn_fused_rank_image_bytes(seg, C, CI);
}

cudaError_t launch_segn_fused(const FusedSegArgs &a, int seg, int C, int units_grid, cudaStream_t stream, bool pdl) {
    using Fn = void (*)(FusedSegArgs);
    Fn fn = nullptr;
    const bool gn = a.gn != 0;
#define SEGN_PICK(S_, C_, H_, G_, P_) \
    if (seg == S_ && C == C_) fn = gn ? segn_fused_kernel<C_, H_, G_, P_, true> : segn_fused_kernel<C_, H_, G_, P_, false>;
    SEGN_PICK(1, 32, 16, 1, 1)
    SEGN_PICK(1, 64, 16, 1, 1)
    SEGN_PICK(2, 64, 8, 2, 1)
    SEGN_PICK(2, 128, 8, 2, 2)
    SEGN_PICK(3, 64, 4, 8, 2)
    SEGN_PICK(3, 128, 4, 8, 4)
#undef SEGN_PICK
    if (!fn) return cudaErrorInvalidValue;
    const size_t smem = segn_fused_smem_bytes(seg, C, a.CI, gn);
    if (!smem) return cudaErrorInvalidValue;
    const int P = segn_fused_cluster(seg, C);
    FusedSegArgs args = a;
    args.smem_budget = 227u * 1024u - 1024u;   // the same budget segn_fused_smem_bytes laid the ring out for
    args.wimg_rank_bytes = segn_fused_rank_image_bytes(seg, C, a.CI);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(units_grid * P);
    cfg.blockDim = dim3(kFnThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = P;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, fn, args);
}

// Builds the fused weight image of one (segment, r_prev, r): per rank p (output rows [p*R, (p+1)*R)),
// the slabs of b0c1, b0c2, the projection, b1c1, b1c2 in consumption order, each [taps][R rows][row
// bytes] K-major and swizzled exactly as the kernel's ring slot expects (swizzle row index relative to
// the 1 KiB-aligned slab start).
namespace {
__global__ void fused_image_kernel(uint8_t *img, const uint16_t *w0, const uint16_t *w1, const uint16_t *wp,
                                   const uint16_t *w3, const uint16_t *w4, int C, int R, int co_off, int CI,
                                   int cin0_full, int cf_full) {
    const bool tapm = 3 * R > 256;
    const int rbi = 2 * fn_ck(CI), rbc = 2 * fn_ck(C);
    const int nchi = (CI + 63) / 64, nchc = (C + 63) / 64;
    const long l1 = static_cast<long>(9) * nchi * R * rbi / 16;   // pieces of L1
    const long l2 = static_cast<long>(9) * nchc * R * rbc / 16;   // pieces of one stride-1 conv
    const long lp = static_cast<long>(nchi) * R * rbi / 16;       // pieces of the projection
    const long total_pieces = l1 + lp + 3 * l2;
    for (long gi = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; gi < total_pieces;
         gi += static_cast<long>(gridDim.x) * blockDim.x) {
        long rem = gi;
        size_t off;
        const uint16_t *w;
        int cin_full, cin_act, taps_k, rb, ch, kh, kw, row_in_slab, piece;
        if (rem < l1) {   // L1: groups (ch, kh in 0,2,1), taps kw 0,2,1
            const int per_kh = 3 * R * rbi / 16;
            const int grp = static_cast<int>(rem / per_kh), r2 = static_cast<int>(rem % per_kh);
            ch = grp / 3;
            const int o = grp % 3;
            kh = o == 0 ? 0 : (o == 1 ? 2 : 1);
            const int tap_i = r2 / (R * rbi / 16), r3 = r2 % (R * rbi / 16);
            kw = tap_i == 0 ? 0 : (tap_i == 1 ? 2 : 1);
            row_in_slab = (tapm ? 0 : tap_i * R) + r3 / (rbi / 16);
            piece = r3 % (rbi / 16);
            off = static_cast<size_t>(grp) * 3 * R * rbi + (tapm ? static_cast<size_t>(tap_i) * R * rbi : 0);
            w = w0;
            cin_full = cin0_full;
            cin_act = CI;
            taps_k = 9;
            rb = rbi;
        } else if (rem - l1 >= l2 && rem - l1 < l2 + lp) {   // projection: chunks, R rows x rbi
            rem -= l1 + l2;
            const int per = R * rbi / 16;
            ch = static_cast<int>(rem / per);
            const int r3 = static_cast<int>(rem % per);
            row_in_slab = r3 / (rbi / 16);
            piece = r3 % (rbi / 16);
            off = static_cast<size_t>(l1 + l2) * 16 + static_cast<size_t>(ch) * R * rbi;
            w = wp;
            cin_full = cin0_full;
            cin_act = CI;
            taps_k = 1;
            rb = rbi;
            kh = kw = 0;
        } else {          // stride-1 convs b0c2 (after L1), b1c1, b1c2 (after the projection)
            rem -= l1;
            int layer;
            size_t base;
            if (rem < l2) {
                layer = 1;
                base = static_cast<size_t>(l1) * 16;
            } else {
                rem -= l2 + lp;
                layer = rem < l2 ? 3 : 4;
                if (layer == 4) rem -= l2;
                base = static_cast<size_t>(l1 + l2 + lp + (layer == 4 ? l2 : 0)) * 16;
            }
            const int per_kh = 3 * R * rbc / 16;
            const int grp = static_cast<int>(rem / per_kh), r2 = static_cast<int>(rem % per_kh);
            ch = grp / 3;
            kh = grp % 3;
            const int tap_i = r2 / (R * rbc / 16), r3 = r2 % (R * rbc / 16);
            kw = tap_i;
            row_in_slab = (tapm ? 0 : tap_i * R) + r3 / (rbc / 16);
            piece = r3 % (rbc / 16);
            off = base + static_cast<size_t>(grp) * 3 * R * rbc + (tapm ? static_cast<size_t>(tap_i) * R * rbc : 0);
            w = layer == 1 ? w1 : (layer == 3 ? w3 : w4);
            cin_full = cf_full;
            cin_act = C;
            taps_k = 9;
            rb = rbc;
        }
        const int co = co_off + row_in_slab % R;
        const int ci0 = ch * 64 + piece * 8;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (ci0 < cin_act)   // channels past the active input width are never multiplied (K steps stop there)
            v = *reinterpret_cast<const uint4 *>(w + (static_cast<size_t>(co) * taps_k + (kh * 3 + kw) * (taps_k == 9)) *
                                                         cin_full + ci0);
        *reinterpret_cast<uint4 *>(img + off + swz_off(row_in_slab, piece, rb)) = v;
    }
}
}  // namespace

cudaError_t build_segn_fused_image(void *img, const void *w0, const void *w1, const void *wp, const void *w3,
                                   const void *w4, int seg, int C, int CI, int cin0_full, int cf_full, cudaStream_t st) {
    const int P = segn_fused_cluster(seg, C), R = C / P;
    const size_t per = segn_fused_rank_image_bytes(seg, C, CI);
    for (int p = 0; p < P; ++p) {
        fused_image_kernel<<<64, 256, 0, st>>>(static_cast<uint8_t *>(img) + p * per, static_cast<const uint16_t *>(w0),
                                               static_cast<const uint16_t *>(w1), static_cast<const uint16_t *>(wp),
                                               static_cast<const uint16_t *>(w3), static_cast<const uint16_t *>(w4), C,
                                               R, p * R, CI, cin0_full, cf_full);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace slim
