// kernels_simt.cu -- the CUDA-core kernels of the hot path.
//
//  * stem: conv3x3 3->c0 + BN + ReLU.  K = 27, arithmetic intensity
//    ~25 FLOP/B: HBM-bound, and a 6-byte pixel stride is not TMA-addressable, so
//    it is a direct conv with the weights and a halo'd input tile in shared memory
//    and 16-byte vector stores (8 output channels per thread).
//  * head: global average pool over the 4x4 map + FC c3 -> classes,
//    fp32 logits.  One CTA per image; pooled vector in smem; one warp per class
//    group with a warp-shuffle dot product.
//  * gather: 16-byte vectorised, coalesced row gather for the packer.
//  * FP32 mode ("FP32/TF32-off"): a register-tiled direct conv with the
//    same three fused epilogues, plain FFMA (tcgen05 has no fp32-input kind).
#include "slim_internal.h"

#include <cuda_bf16.h>

#include <algorithm>

namespace slim {
namespace {

__device__ __forceinline__ float bf16_to_f(uint16_t h) { return __uint_as_float(static_cast<uint32_t>(h) << 16); }
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t *>(&h);
}

template <typename T> __device__ __forceinline__ float ld_act(const T *p);
template <> __device__ __forceinline__ float ld_act<uint16_t>(const uint16_t *p) { return bf16_to_f(*p); }
template <> __device__ __forceinline__ float ld_act<float>(const float *p) { return *p; }

// ---------------------------------------------------------------- stem
// Block: one image x kStemRows output rows, all W columns.  Threads map to
// (pixel, group of 8 output channels) so consecutive threads store consecutive
// 16-byte (bf16) / 32-byte (fp32) pieces: fully coalesced.
constexpr int kStemRows = 4;
constexpr int kStemThreads = 256;
constexpr int kMaxStemW = 64, kMaxStemC = 4, kMaxStemCout = 64;

template <typename TIn, typename TOut>
__global__ void __launch_bounds__(kStemThreads)
    stem_kernel(const TIn *__restrict__ in, const float *__restrict__ w, int cin_full, const float *__restrict__ scale,
                const float *__restrict__ shift, TOut *__restrict__ out, int H, int W, int cimg, int c0,
                float relu_lo) {
    __shared__ float s_in[(kStemRows + 2) * (kMaxStemW + 2) * kMaxStemC];
    __shared__ float s_w[kMaxStemCout * 9 * kMaxStemC];
    const int n = blockIdx.y;
    const int h0 = blockIdx.x * kStemRows;
    const int TW = W + 2;
    // halo'd input tile rows h0-1 .. h0+kStemRows, cols -1 .. W (zero padded)
    for (int i = threadIdx.x; i < (kStemRows + 2) * TW * cimg; i += blockDim.x) {
        const int c = i % cimg, col = (i / cimg) % TW, r = i / (cimg * TW);
        const int ih = h0 + r - 1, iw = col - 1;
        float v = 0.f;
        if (ih >= 0 && ih < H && iw >= 0 && iw < W) v = ld_act(in + ((static_cast<size_t>(n) * H + ih) * W + iw) * cimg + c);
        s_in[i] = v;
    }
    for (int i = threadIdx.x; i < c0 * 9 * cimg; i += blockDim.x) {
        const int ci = i % cimg, tap = (i / cimg) % 9, co = i / (9 * cimg);
        s_w[i] = w[(static_cast<size_t>(co) * 9 + tap) * cin_full + ci];
    }
    __syncthreads();
    const int groups = c0 / 8;
    const int items = kStemRows * W * groups;
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
        const int g = it % groups, pix = it / groups;
        const int r = pix / W, col = pix % W;
        if (h0 + r >= H) continue;
        float acc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = 0.f;
        for (int kh = 0; kh < 3; ++kh)
            for (int kw = 0; kw < 3; ++kw)
                for (int ci = 0; ci < cimg; ++ci) {
                    const float x = s_in[((r + kh) * TW + col + kw) * cimg + ci];
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[j] = fmaf(x, s_w[((g * 8 + j) * 9 + kh * 3 + kw) * cimg + ci], acc[j]);
                }
        const size_t o = ((static_cast<size_t>(n) * H + h0 + r) * W + col) * c0 + g * 8;
        float y[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) y[j] = fmaxf(fmaf(acc[j], scale[g * 8 + j], shift[g * 8 + j]), relu_lo);
        if constexpr (sizeof(TOut) == 2) {
            uint4 v = make_uint4(pack2(y[0], y[1]), pack2(y[2], y[3]), pack2(y[4], y[5]), pack2(y[6], y[7]));
            *reinterpret_cast<uint4 *>(out + o) = v;
        } else {
            *reinterpret_cast<float4 *>(out + o) = make_float4(y[0], y[1], y[2], y[3]);
            *reinterpret_cast<float4 *>(out + o + 4) = make_float4(y[4], y[5], y[6], y[7]);
        }
    }
}

// ---------------------------------------------------------------- head
// Grid (ceil(B/8), ceil(K/kHeadClasses)).  A CTA pools its 8 images into smem
// (fp32; 16 independent loads in flight per thread), then each warp takes classes
// k of its group; each lane holds its slice of the FC row in registers (all loads
// issued before the FMAs) and accumulates the 8 images at once; warp-shuffle sum.
constexpr int kHeadThreads = 256;
constexpr int kHeadImgs = 8;
constexpr int kHeadClasses = 16;
constexpr int kHeadMaxC = 1024;   // c3 <= 1024 -> <= 32 channels per lane
template <typename TIn>
__global__ void __launch_bounds__(kHeadThreads)
    head_kernel(const TIn *__restrict__ in, const float *__restrict__ fc_w, const float *__restrict__ fc_b,
                float *__restrict__ logits, int B, int P, int c3, int c3_full, int K) {
    extern __shared__ float s_p[];   // [kHeadImgs][c3]
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int n0 = blockIdx.x * kHeadImgs;
    const int ni = min(kHeadImgs, B - n0);
    const float inv = 1.f / static_cast<float>(P);
    for (int i = threadIdx.x; i < kHeadImgs * c3; i += blockDim.x) {   // consecutive threads: consecutive channels
        const int img = i / c3, c = i - img * c3;
        float sum = 0.f;
        if (img < ni) {
            const TIn *x = in + (static_cast<size_t>(n0 + img) * P) * c3 + c;
            int p = 0;
            for (; p + 8 <= P; p += 8) {
                float v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = ld_act(x + static_cast<size_t>(p + u) * c3);
#pragma unroll
                for (int u = 0; u < 8; ++u) sum += v[u];
            }
            for (; p < P; ++p) sum += ld_act(x + static_cast<size_t>(p) * c3);
        }
        s_p[i] = sum * inv;
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int k_end = min(K, (blockIdx.y + 1) * kHeadClasses);
    for (int k = blockIdx.y * kHeadClasses + warp; k < k_end; k += nw) {
        const float *wr = fc_w + static_cast<size_t>(k) * c3_full;
        float w[kHeadMaxC / 32];
#pragma unroll
        for (int i = 0; i < kHeadMaxC / 32; ++i) {
            const int c = lane + 32 * i;
            w[i] = (c < c3) ? __ldg(wr + c) : 0.f;
        }
        float d[kHeadImgs];
#pragma unroll
        for (int j = 0; j < kHeadImgs; ++j) d[j] = 0.f;
#pragma unroll
        for (int i = 0; i < kHeadMaxC / 32; ++i) {
            const int c = lane + 32 * i;
            if (c < c3) {
#pragma unroll
                for (int j = 0; j < kHeadImgs; ++j) d[j] = fmaf(s_p[j * c3 + c], w[i], d[j]);
            }
        }
#pragma unroll
        for (int j = 0; j < kHeadImgs; ++j)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) d[j] += __shfl_xor_sync(0xffffffffu, d[j], o);
        if (lane < ni) {
            float v = d[0];
#pragma unroll
            for (int j = 1; j < kHeadImgs; ++j) v = (lane == j) ? d[j] : v;
            logits[static_cast<size_t>(n0 + lane) * K + k] = v + fc_b[k];
        }
    }
}

// FC on pooled fp32 features (global average pool fused into the last conv's
// epilogue): grid (ceil(B/8), ceil(K/16)); the 8 pooled vectors are loaded with
// independent 16-byte loads, each FC row is held in registers, warp-shuffle sums.
__global__ void __launch_bounds__(kHeadThreads)
    fc_kernel(const float *__restrict__ pooled, const float *__restrict__ fc_w, const float *__restrict__ fc_b,
              float *__restrict__ logits, int B, int c3, int c3_full, int K) {
    extern __shared__ float s_p[];   // [kHeadImgs][c3]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int k0 = blockIdx.y * kHeadClasses + warp, k1 = k0 + nw;   // kHeadClasses == 2 * warps
    // FC rows are weights (not produced by the previous kernel): load them before the PDL wait
    float w0[kHeadMaxC / 32], w1[kHeadMaxC / 32];
#pragma unroll
    for (int i = 0; i < kHeadMaxC / 32; ++i) {
        const int c = lane + 32 * i;
        w0[i] = (c < c3 && k0 < K) ? __ldg(fc_w + static_cast<size_t>(k0) * c3_full + c) : 0.f;
        w1[i] = (c < c3 && k1 < K) ? __ldg(fc_w + static_cast<size_t>(k1) * c3_full + c) : 0.f;
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int n0 = blockIdx.x * kHeadImgs;
    const int ni = min(kHeadImgs, B - n0);
    const int nv = ni * c3 / 4;
    const float4 *src = reinterpret_cast<const float4 *>(pooled + static_cast<size_t>(n0) * c3);
    for (int i = threadIdx.x; i < kHeadImgs * c3 / 4; i += blockDim.x)
        reinterpret_cast<float4 *>(s_p)[i] = i < nv ? __ldg(src + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    __syncthreads();
    float d0[kHeadImgs], d1[kHeadImgs];
#pragma unroll
    for (int j = 0; j < kHeadImgs; ++j) d0[j] = d1[j] = 0.f;
#pragma unroll
    for (int i = 0; i < kHeadMaxC / 32; ++i) {
        const int c = lane + 32 * i;
        if (c < c3) {
#pragma unroll
            for (int j = 0; j < kHeadImgs; ++j) {
                const float p = s_p[j * c3 + c];
                d0[j] = fmaf(p, w0[i], d0[j]);
                d1[j] = fmaf(p, w1[i], d1[j]);
            }
        }
    }
#pragma unroll
    for (int j = 0; j < kHeadImgs; ++j)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            d0[j] += __shfl_xor_sync(0xffffffffu, d0[j], o);
            d1[j] += __shfl_xor_sync(0xffffffffu, d1[j], o);
        }
    if (lane < ni) {
        float v0 = d0[0], v1 = d1[0];
#pragma unroll
        for (int j = 1; j < kHeadImgs; ++j) {
            v0 = (lane == j) ? d0[j] : v0;
            v1 = (lane == j) ? d1[j] : v1;
        }
        if (k0 < K) logits[static_cast<size_t>(n0 + lane) * K + k0] = v0 + fc_b[k0];
        if (k1 < K) logits[static_cast<size_t>(n0 + lane) * K + k1] = v1 + fc_b[k1];
    }
}

// ---------------------------------------------------------------- gather
__global__ void gather_kernel(const uint4 *__restrict__ src, size_t src_stride, const uint32_t *__restrict__ idx, int n,
                              size_t per_row, uint4 *__restrict__ dst) {
    const size_t total = static_cast<size_t>(n) * per_row;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t r = i / per_row, off = i - r * per_row;
        dst[i] = __ldg(src + static_cast<size_t>(idx[r]) * src_stride + off);
    }
}

// scatter (inverse of gather): dst + idx[r]*dst_stride <- src row r
__global__ void scatter_kernel(const uint4 *__restrict__ src, const uint32_t *__restrict__ idx, int n, size_t per_row,
                               uint4 *__restrict__ dst, size_t dst_stride) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const size_t total = static_cast<size_t>(n) * per_row;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t r = i / per_row, off = i - r * per_row;
        dst[static_cast<size_t>(idx[r]) * dst_stride + off] = __ldg(src + i);
    }
}

// ---------------------------------------------------------------- FP32 conv
// One thread computes 4 output pixels (along W) x 4 output channels; weights
// for the CTA's 32 output channels of one tap-chunk are staged in smem.
constexpr int kF32Threads = 128;
__global__ void __launch_bounds__(kF32Threads) conv_f32_kernel(const ConvF32Args a) {
    const int co_base = blockIdx.y * 32;
    const int tid = threadIdx.x;
    const int cq = tid & 7;            // channel quad: co_base + 4*cq .. +3
    const int pg = tid >> 3;           // pixel group (16 per CTA), 4 pixels each
    const long pix0 = (static_cast<long>(blockIdx.x) * 16 + pg) * 4;
    const long npix = static_cast<long>(a.B) * a.Ho * a.Wo;
    float acc[4][4], acc1[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = acc1[i][j] = 0.f;
    int pn[4], poh[4], pow_[4];
    bool pv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const long p = pix0 + i;
        pv[i] = p < npix;
        const long pp = pv[i] ? p : 0;
        pn[i] = static_cast<int>(pp / (a.Ho * a.Wo));
        poh[i] = static_cast<int>((pp / a.Wo) % a.Ho);
        pow_[i] = static_cast<int>(pp % a.Wo);
    }
    const int co = co_base + cq * 4;
    for (int part = 0; part < (a.epi == EPI_BN_PROJ_RELU ? 2 : 1); ++part) {
        const float *x = part ? a.x1 : a.x;
        const float *w = part ? a.w1 : a.w;
        const int H = part ? a.H1 : a.H, W = part ? a.W1 : a.W, cin = part ? a.c_in1 : a.c_in;
        const int k = part ? 1 : a.k, st = part ? a.stride1 : a.stride, pad = part ? 0 : a.pad;
        const int cin_full = part ? a.cin1_full : a.cin_full;
        float(*ac)[4] = part ? acc1 : acc;
        for (int kh = 0; kh < k; ++kh)
            for (int kw = 0; kw < k; ++kw) {
                const float *xr[4];
                bool ok[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int ih = st * poh[i] + kh - pad, iw = st * pow_[i] + kw - pad;
                    ok[i] = pv[i] && ih >= 0 && ih < H && iw >= 0 && iw < W;
                    xr[i] = x + ((static_cast<size_t>(pn[i]) * H + (ok[i] ? ih : 0)) * W + (ok[i] ? iw : 0)) * cin;
                }
                const float *wr[4];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    wr[j] = w + ((static_cast<size_t>(co + j < a.c_out ? co + j : 0) * k + kh) * k + kw) * cin_full;
                for (int ci = 0; ci < cin; ++ci) {
                    float xv[4], wv[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) xv[i] = ok[i] ? __ldg(xr[i] + ci) : 0.f;
#pragma unroll
                    for (int j = 0; j < 4; ++j) wv[j] = __ldg(wr[j] + ci);
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) ac[i][j] = fmaf(xv[i], wv[j], ac[i][j]);
                }
            }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (!pv[i]) continue;
        const size_t o = static_cast<size_t>(pix0 + i) * a.c_out;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int c = co + j;
            if (c >= a.c_out) continue;
            float f = fmaf(acc[i][j], a.scale0[c], a.shift0[c]);
            if (a.epi == EPI_BN_PROJ_RELU) f += fmaf(acc1[i][j], a.scale1[c], a.shift1[c]);
            if (a.epi == EPI_BN_ADD_RELU) f += a.res[o + c];
            a.out[o + c] = fmaxf(f, a.relu_lo);
        }
    }
}

// FP32 implicit GEMM: CTA tile 128 output pixels x 64 output channels, K in steps of
// 16 input channels of one tap, double-buffered through shared memory (A stored k-major so a
// thread reads its 8 pixels as two float4, B as one float4 of 4 channels); each thread owns an
// 8 x 4 register tile (32 FFMA per 3 LDS.128).  Same fused epilogues as conv_f32_kernel.
constexpr int kGM = 128, kGN = 64, kGK = 16, kGThreads = 256;

struct GemmTile {   // per-thread loader / compute coordinates of conv_f32_gemm_kernel
    int tx, ty, lp, lc, lb, lbc, pn, poh, pw, gco;
    bool pok, cok;
};

// acc += the GEMM of one conv part (K = k*k*cin in steps of 16 channels of one tap)
__device__ __forceinline__ void f32_gemm_part(const GemmTile &g, const float *__restrict__ x, const float *__restrict__ w,
                                              int H, int W, int cin, int k, int st, int pad, int cin_full,
                                              float (*As)[kGK][kGM + 4], float (*Bs)[kGK][kGN + 4], float (&acc)[8][4],
                                              int split = 0, int nsplit = 1) {
    const int csteps = cin / kGK, steps_all = k * k * csteps;
    // split-K: this CTA's consecutive range of the K steps (the whole range when nsplit == 1)
    const int s_lo = steps_all * split / nsplit, steps = steps_all * (split + 1) / nsplit - s_lo;
    float4 ra0, ra1, rb;
    auto load = [&](int s) {
        s += s_lo;
        const int tap = s / csteps, c0 = (s - tap * csteps) * kGK, kh = tap / k, kw = tap - kh * k;
        const int ih = st * g.poh + kh - pad, iw = st * g.pw + kw - pad;
        const bool ok = g.pok && ih >= 0 && ih < H && iw >= 0 && iw < W;
        const float *xp = x + ((static_cast<size_t>(g.pn) * H + (ok ? ih : 0)) * W + (ok ? iw : 0)) * cin + c0 + g.lc;
        ra0 = ok ? __ldg(reinterpret_cast<const float4 *>(xp)) : make_float4(0.f, 0.f, 0.f, 0.f);
        ra1 = ok ? __ldg(reinterpret_cast<const float4 *>(xp + 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
        const float *wp = w + ((static_cast<size_t>(g.cok ? g.gco : 0) * k + kh) * k + kw) * cin_full + c0 + g.lbc;
        rb = g.cok ? __ldg(reinterpret_cast<const float4 *>(wp)) : make_float4(0.f, 0.f, 0.f, 0.f);
    };
    auto store = [&](int b) {
        As[b][g.lc + 0][g.lp] = ra0.x;
        As[b][g.lc + 1][g.lp] = ra0.y;
        As[b][g.lc + 2][g.lp] = ra0.z;
        As[b][g.lc + 3][g.lp] = ra0.w;
        As[b][g.lc + 4][g.lp] = ra1.x;
        As[b][g.lc + 5][g.lp] = ra1.y;
        As[b][g.lc + 6][g.lp] = ra1.z;
        As[b][g.lc + 7][g.lp] = ra1.w;
        Bs[b][g.lbc + 0][g.lb] = rb.x;
        Bs[b][g.lbc + 1][g.lb] = rb.y;
        Bs[b][g.lbc + 2][g.lb] = rb.z;
        Bs[b][g.lbc + 3][g.lb] = rb.w;
    };
    __syncthreads();   // a previous part's last tile has been consumed
    load(0);
    store(0);
    __syncthreads();
#pragma unroll 1
    for (int s = 0; s < steps; ++s) {
        const int b = s & 1;
        if (s + 1 < steps) load(s + 1);
#pragma unroll
        for (int kk = 0; kk < kGK; ++kk) {
            // pixels tx*4 .. +3 and kGM/2 + tx*4 .. +3: each LDS.128 of the warp reads one contiguous run
            // (tx*8 .. +7 put the lanes 32 B apart: two bank wavefronts per 128 B, ncu: 40 % of the
            // shared-load wavefronts were conflicts)
            const float4 a0 = *reinterpret_cast<const float4 *>(&As[b][kk][g.tx * 4]);
            const float4 a1 = *reinterpret_cast<const float4 *>(&As[b][kk][kGM / 2 + g.tx * 4]);
            const float4 bv = *reinterpret_cast<const float4 *>(&Bs[b][kk][g.ty * 4]);
            const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float bw[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bw[j], acc[i][j]);
        }
        if (s + 1 < steps) store(b ^ 1);
        __syncthreads();
    }
}

__device__ __forceinline__ void conv_f32_gemm_tile(const ConvF32Args &a, int bx, int by, int split = 0) {
    __shared__ __align__(16) float As[2][kGK][kGM + 4];
    __shared__ __align__(16) float Bs[2][kGK][kGN + 4];
    const int tid = threadIdx.x;
    const long m0 = static_cast<long>(bx) * kGM;
    const int n0 = by * kGN;
    const long npix = static_cast<long>(a.B) * a.Ho * a.Wo;
    GemmTile g;
    g.tx = tid & 15;          // compute: pixels tx*4 .. +3 and 64 + tx*4 .. +3, channels ty*4 .. +3
    g.ty = tid >> 4;
    g.lp = tid >> 1;          // A loader: pixel lp, channels lc .. lc+7 of the 16-channel step
    g.lc = (tid & 1) * 8;
    g.lb = tid >> 2;          // B loader: channel lb, ci lbc .. lbc+3
    g.lbc = (tid & 3) * 4;
    const long gp = m0 + g.lp;
    g.pok = gp < npix;
    const long gpp = g.pok ? gp : 0;
    g.pn = static_cast<int>(gpp / (a.Ho * a.Wo));
    g.poh = static_cast<int>((gpp / a.Wo) % a.Ho);
    g.pw = static_cast<int>(gpp % a.Wo);
    g.gco = n0 + g.lb;
    g.cok = g.gco < a.c_out;
    const int tx = g.tx, ty = g.ty;
    float acc0[8][4], acc1[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc0[i][j] = acc1[i][j] = 0.f;
    const int nparts = a.epi == EPI_BN_PROJ_RELU ? 2 : 1;
    const int ks = a.ksplit > 1 ? a.ksplit : 1;
    f32_gemm_part(g, a.x, a.w, a.H, a.W, a.c_in, a.k, a.stride, a.pad, a.cin_full, As, Bs, acc0, split, ks);
    // (split-K: the projection shortcut is computed whole by split 0, into its own partial slot ks)
    const bool do_proj = nparts == 2 && split == 0;
    if (do_proj) f32_gemm_part(g, a.x1, a.w1, a.H1, a.W1, a.c_in1, 1, a.stride1, 0, a.cin1_full, As, Bs, acc1);
    const int c = n0 + ty * 4;
    if (c >= a.c_out) return;   // c_out is a multiple of 16: a thread's 4 channels are all valid or none
    if (ks > 1) {   // raw partial sums of this K range; conv_f32_splitk_reduce applies the epilogue
        float *dst = a.part + static_cast<size_t>(split) * npix * a.c_out;
        float *dstp = a.part + static_cast<size_t>(ks) * npix * a.c_out;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const long p = m0 + (i < 4 ? tx * 4 + i : kGM / 2 + tx * 4 + i - 4);
            if (p < npix) {
                *reinterpret_cast<float4 *>(dst + static_cast<size_t>(p) * a.c_out + c) =
                    make_float4(acc0[i][0], acc0[i][1], acc0[i][2], acc0[i][3]);
                if (do_proj)
                    *reinterpret_cast<float4 *>(dstp + static_cast<size_t>(p) * a.c_out + c) =
                        make_float4(acc1[i][0], acc1[i][1], acc1[i][2], acc1[i][3]);
            }
        }
        return;
    }
    const float4 s0 = *reinterpret_cast<const float4 *>(a.scale0 + c), t0 = *reinterpret_cast<const float4 *>(a.shift0 + c);
    float4 s1 = make_float4(0.f, 0.f, 0.f, 0.f), t1 = s1;
    if (nparts == 2) {
        s1 = *reinterpret_cast<const float4 *>(a.scale1 + c);
        t1 = *reinterpret_cast<const float4 *>(a.shift1 + c);
    }
    const float sc0[4] = {s0.x, s0.y, s0.z, s0.w}, sh0[4] = {t0.x, t0.y, t0.z, t0.w};
    const float sc1[4] = {s1.x, s1.y, s1.z, s1.w}, sh1[4] = {t1.x, t1.y, t1.z, t1.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const long p = m0 + (i < 4 ? tx * 4 + i : kGM / 2 + tx * 4 + i - 4);
        if (p >= npix) continue;
        const size_t o = static_cast<size_t>(p) * a.c_out + c;
        float r[4] = {0.f, 0.f, 0.f, 0.f};
        if (a.epi == EPI_BN_ADD_RELU) {
            const float4 rv = *reinterpret_cast<const float4 *>(a.res + o);
            r[0] = rv.x;
            r[1] = rv.y;
            r[2] = rv.z;
            r[3] = rv.w;
        }
        float f[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            f[j] = fmaf(acc0[i][j], sc0[j], sh0[j]);
            if (nparts == 2) f[j] += fmaf(acc1[i][j], sc1[j], sh1[j]);
            f[j] = fmaxf(f[j] + r[j], a.relu_lo);
        }
        *reinterpret_cast<float4 *>(a.out + o) = make_float4(f[0], f[1], f[2], f[3]);
    }
}

// persistent over (M tile, N tile): the grid may be capped (SM share of the width, max_ctas)
__global__ void __launch_bounds__(kGThreads) conv_f32_gemm_kernel(const ConvF32Args a, int gx, int gy) {
    const int ks = a.ksplit > 1 ? a.ksplit : 1;
    for (int t = blockIdx.x; t < gx * gy * ks; t += gridDim.x) {
        const int tt = t % (gx * gy);
        conv_f32_gemm_tile(a, tt % gx, tt / gx, t / (gx * gy));
        __syncthreads();
    }
}

// Wider variant for layers without a projection: CTA tile 256 pixels x 64 channels, 8 x 8 register
// tile per thread (64 FFMA per 4 LDS.128).
constexpr int kWM = 256;
__device__ __forceinline__ void conv_f32_gemm256_tile(const ConvF32Args &a, int bx, int by) {
    __shared__ __align__(16) float As[2][kGK][kWM + 4];
    __shared__ __align__(16) float Bs[2][kGK][kGN + 4];
    const int tid = threadIdx.x;
    const int tx = tid & 31, ty = tid >> 5;       // compute: pixels tx*4 .. +3, 128 + tx*4 .. +3; channels ty*8 .. +7
    const long m0 = static_cast<long>(bx) * kWM;
    const int n0 = by * kGN;
    const long npix = static_cast<long>(a.B) * a.Ho * a.Wo;
    const long gp = m0 + tid;                      // A loader: one pixel, 16 channels
    const bool pok = gp < npix;
    const long gpp = pok ? gp : 0;
    const int pn = static_cast<int>(gpp / (a.Ho * a.Wo)), poh = static_cast<int>((gpp / a.Wo) % a.Ho),
              pw = static_cast<int>(gpp % a.Wo);
    const int lb = tid >> 2, lbc = (tid & 3) * 4;  // B loader: channel lb, ci lbc .. +3
    const int gco = n0 + lb;
    const bool cok = gco < a.c_out;
    const int H = a.H, W = a.W, cin = a.c_in, k = a.k, st = a.stride, pad = a.pad;
    const int csteps = cin / kGK, steps = k * k * csteps;
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    float4 ra[4], rb;
    auto load = [&](int s) {
        const int tap = s / csteps, c0 = (s - tap * csteps) * kGK, kh = tap / k, kw = tap - kh * k;
        const int ih = st * poh + kh - pad, iw = st * pw + kw - pad;
        const bool ok = pok && ih >= 0 && ih < H && iw >= 0 && iw < W;
        const float *xp = a.x + ((static_cast<size_t>(pn) * H + (ok ? ih : 0)) * W + (ok ? iw : 0)) * cin + c0;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            ra[q] = ok ? __ldg(reinterpret_cast<const float4 *>(xp) + q) : make_float4(0.f, 0.f, 0.f, 0.f);
        const float *wp = a.w + ((static_cast<size_t>(cok ? gco : 0) * k + kh) * k + kw) * a.cin_full + c0 + lbc;
        rb = cok ? __ldg(reinterpret_cast<const float4 *>(wp)) : make_float4(0.f, 0.f, 0.f, 0.f);
    };
    auto store = [&](int b) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            As[b][4 * q + 0][tid] = ra[q].x;
            As[b][4 * q + 1][tid] = ra[q].y;
            As[b][4 * q + 2][tid] = ra[q].z;
            As[b][4 * q + 3][tid] = ra[q].w;
        }
        Bs[b][lbc + 0][lb] = rb.x;
        Bs[b][lbc + 1][lb] = rb.y;
        Bs[b][lbc + 2][lb] = rb.z;
        Bs[b][lbc + 3][lb] = rb.w;
    };
    load(0);
    store(0);
    __syncthreads();
#pragma unroll 1
    for (int s = 0; s < steps; ++s) {
        const int b = s & 1;
        if (s + 1 < steps) load(s + 1);
#pragma unroll
        for (int kk = 0; kk < kGK; ++kk) {
            const float4 a0 = *reinterpret_cast<const float4 *>(&As[b][kk][tx * 4]);   // conflict-free runs
            const float4 a1 = *reinterpret_cast<const float4 *>(&As[b][kk][kWM / 2 + tx * 4]);
            const float4 b0 = *reinterpret_cast<const float4 *>(&Bs[b][kk][ty * 8]);
            const float4 b1 = *reinterpret_cast<const float4 *>(&Bs[b][kk][ty * 8 + 4]);
            const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float bw[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bw[j], acc[i][j]);
        }
        if (s + 1 < steps) store(b ^ 1);
        __syncthreads();
    }
    const int c = n0 + ty * 8;
    if (c >= a.c_out) return;   // c_out is a multiple of 16: a thread's 8 channels are all valid or none
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const long p = m0 + (i < 4 ? tx * 4 + i : kWM / 2 + tx * 4 + i - 4);
        if (p >= npix) continue;
        const size_t o = static_cast<size_t>(p) * a.c_out + c;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            float f[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int cc = c + 4 * h + j;
                f[j] = fmaf(acc[i][4 * h + j], a.scale0[cc], a.shift0[cc]);
                if (a.epi == EPI_BN_ADD_RELU) f[j] += a.res[o + 4 * h + j];
                f[j] = fmaxf(f[j], a.relu_lo);
            }
            *reinterpret_cast<float4 *>(a.out + o + 4 * h) = make_float4(f[0], f[1], f[2], f[3]);
        }
    }
}

__global__ void __launch_bounds__(kGThreads, 1) conv_f32_gemm256_kernel(const ConvF32Args a, int gx, int gy) {
    for (int t = blockIdx.x; t < gx * gy; t += gridDim.x) {
        conv_f32_gemm256_tile(a, t % gx, t / gx);
        __syncthreads();
    }
}

}  // namespace

cudaError_t launch_stem_bf16(const uint16_t *in, const float *w, int cin_full, const float *scale, const float *shift,
                             uint16_t *out, int B, int H, int W, int cimg, int c0, cudaStream_t s,
                             float relu_lo) {
    if (W > kMaxStemW || cimg > kMaxStemC || c0 > kMaxStemCout || c0 % 8) return cudaErrorInvalidValue;
    dim3 grid((H + kStemRows - 1) / kStemRows, B);
    stem_kernel<uint16_t, uint16_t><<<grid, kStemThreads, 0, s>>>(in, w, cin_full, scale, shift, out, H, W, cimg, c0, relu_lo);
    return cudaGetLastError();
}
cudaError_t launch_stem_f32(const float *in, const float *w, int cin_full, const float *scale, const float *shift,
                            float *out, int B, int H, int W, int cimg, int c0, cudaStream_t s,
                            float relu_lo) {
    if (W > kMaxStemW || cimg > kMaxStemC || c0 > kMaxStemCout || c0 % 8) return cudaErrorInvalidValue;
    dim3 grid((H + kStemRows - 1) / kStemRows, B);
    stem_kernel<float, float><<<grid, kStemThreads, 0, s>>>(in, w, cin_full, scale, shift, out, H, W, cimg, c0, relu_lo);
    return cudaGetLastError();
}
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl,
                       Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

cudaError_t launch_head_bf16(const uint16_t *in, const float *fc_w, const float *fc_b, float *logits, int B, int P,
                             int c3, int c3_full, int K, cudaStream_t s, bool pdl) {
    return launch_pdl(head_kernel<uint16_t>,
                      dim3((B + kHeadImgs - 1) / kHeadImgs, (K + kHeadClasses - 1) / kHeadClasses), dim3(kHeadThreads),
                      kHeadImgs * c3 * sizeof(float), s, pdl, in, fc_w, fc_b, logits, B, P, c3, c3_full, K);
}
cudaError_t launch_head_f32(const float *in, const float *fc_w, const float *fc_b, float *logits, int B, int P, int c3,
                            int c3_full, int K, cudaStream_t s, bool pdl) {
    return launch_pdl(head_kernel<float>,
                      dim3((B + kHeadImgs - 1) / kHeadImgs, (K + kHeadClasses - 1) / kHeadClasses), dim3(kHeadThreads),
                      kHeadImgs * c3 * sizeof(float), s, pdl, in, fc_w, fc_b, logits, B, P, c3, c3_full, K);
}
cudaError_t launch_fc_f32(const float *pooled, const float *fc_w, const float *fc_b, float *logits, int B, int c3,
                          int c3_full, int K, cudaStream_t s, bool pdl) {
    if (c3 % 4 || c3 > kHeadMaxC) return cudaErrorInvalidValue;
    return launch_pdl(fc_kernel, dim3((B + kHeadImgs - 1) / kHeadImgs, (K + kHeadClasses - 1) / kHeadClasses),
                      dim3(kHeadThreads), kHeadImgs * c3 * sizeof(float), s, pdl, pooled, fc_w, fc_b, logits, B, c3,
                      c3_full, K);
}
cudaError_t launch_gather(const void *src, size_t src_stride, const uint32_t *idx, int n, size_t row_bytes, void *dst,
                          cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const size_t per_row = row_bytes / 16;
    const size_t total = per_row * n;
    int blocks = static_cast<int>((total + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    gather_kernel<<<blocks, 256, 0, s>>>(static_cast<const uint4 *>(src), src_stride / 16, idx, n, per_row,
                                         static_cast<uint4 *>(dst));
    return cudaGetLastError();
}
cudaError_t launch_scatter(const void *src, const uint32_t *idx, int n, size_t row_bytes, void *dst, size_t dst_stride,
                           cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const size_t per_row = row_bytes / 16;
    const size_t total = per_row * n;
    int blocks = static_cast<int>((total + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    scatter_kernel<<<blocks, 256, 0, s>>>(static_cast<const uint4 *>(src), idx, n, per_row, static_cast<uint4 *>(dst),
                                          dst_stride / 16);
    return cudaGetLastError();
}
// split-K reduce + epilogue: out = max(sum_split part * scale + shift + res, relu_lo), the partials summed
// in split order (one float4 of 4 channels per thread)
__global__ void conv_f32_splitk_reduce(const ConvF32Args a) {
    const size_t npix = static_cast<size_t>(a.B) * a.Ho * a.Wo, n4 = npix * a.c_out / 4;
    for (size_t v = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; v < n4; v += gridDim.x * blockDim.x) {
        const size_t o = v * 4;
        const int c = static_cast<int>(o % a.c_out);
        float4 s = *reinterpret_cast<const float4 *>(a.part + o);
        for (int k = 1; k < a.ksplit; ++k) {
            const float4 q = *reinterpret_cast<const float4 *>(a.part + k * npix * a.c_out + o);
            s.x += q.x;
            s.y += q.y;
            s.z += q.z;
            s.w += q.w;
        }
        float f[4] = {s.x, s.y, s.z, s.w}, r[4] = {0.f, 0.f, 0.f, 0.f};
        if (a.epi == EPI_BN_ADD_RELU) {
            const float4 rv = *reinterpret_cast<const float4 *>(a.res + o);
            r[0] = rv.x;
            r[1] = rv.y;
            r[2] = rv.z;
            r[3] = rv.w;
        }
        if (a.epi == EPI_BN_PROJ_RELU) {   // + the shortcut's BN of its raw projection (slot ksplit)
            const float4 q = *reinterpret_cast<const float4 *>(a.part + a.ksplit * npix * a.c_out + o);
            const float qq[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) r[j] = fmaf(qq[j], a.scale1[c + j], a.shift1[c + j]);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) f[j] = fmaxf(fmaf(f[j], a.scale0[c + j], a.shift0[c + j]) + r[j], a.relu_lo);
        *reinterpret_cast<float4 *>(a.out + o) = make_float4(f[0], f[1], f[2], f[3]);
    }
}

cudaError_t launch_conv_f32(const ConvF32Args &a, cudaStream_t s) {
    const long npix = static_cast<long>(a.B) * a.Ho * a.Wo;
    static const bool direct = getenv("SLIM_F32_DIRECT") != nullptr;   // A/B: the direct-conv kernel
    // the 256 x 64 tile (8 x 8 per thread, 167 registers: one CTA per SM) measured 1.7 % slower than the
    // 128 x 64 tile (8 x 4, two CTAs per SM) once both read A conflict-free: opt-in SLIM_F32_GEMM256=1
    static const bool wide = getenv("SLIM_F32_GEMM256") != nullptr;
    if (!direct && wide && a.c_in % kGK == 0 && a.epi != EPI_BN_PROJ_RELU && a.c_out % 16 == 0 &&
        npix >= 148L * kWM) {
        const int gx = static_cast<int>((npix + kWM - 1) / kWM), gy = (a.c_out + kGN - 1) / kGN;
        const int grid = (a.max_ctas > 0 && a.max_ctas < gx * gy) ? a.max_ctas : gx * gy;
        conv_f32_gemm256_kernel<<<grid, kGThreads, 0, s>>>(a, gx, gy);
        return cudaGetLastError();
    }
    if (!direct && a.c_in % kGK == 0 && (a.epi != EPI_BN_PROJ_RELU || a.c_in1 % kGK == 0) && a.c_out % 16 == 0) {
        const int gx = static_cast<int>((npix + kGM - 1) / kGM), gy = (a.c_out + kGN - 1) / kGN;
        const int ks = (a.ksplit > 1 && a.part) ? a.ksplit : 1;
        ConvF32Args b = a;
        b.ksplit = ks;
        const int work = gx * gy * ks;
        const int grid = (a.max_ctas > 0 && a.max_ctas < work) ? a.max_ctas : work;
        conv_f32_gemm_kernel<<<grid, kGThreads, 0, s>>>(b, gx, gy);
        if (ks > 1) {
            const size_t n4 = static_cast<size_t>(npix) * a.c_out / 4;
            conv_f32_splitk_reduce<<<static_cast<unsigned>(std::min<size_t>((n4 + 255) / 256, 148 * 8)), 256, 0, s>>>(b);
        }
        return cudaGetLastError();
    }
    dim3 grid(static_cast<unsigned>((npix + 63) / 64), (a.c_out + 31) / 32);
    conv_f32_kernel<<<grid, kF32Threads, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace slim
