// kernels_gn.cu -- GroupNorm (+ shortcut) (+ ReLU) for the GroupNorm variant of the network.
//
// "We employ Group Normalization instead of Batch Normalization to avoid
// cross-width statistics drift".  Reading R16: groups of `cpg` (16) consecutive
// channels; statistics per (image, group) over H*W*cpg values; biased variance; eps.
//
// The convs run with an identity epilogue and no ReLU (relu_lo = -inf) and store the raw
// pre-norm output y; this kernel then computes, per (image n, group g),
//   mu = mean(y[n, :, :, g]),  var = mean((y - mu)^2)          (fp32; one pass over registers in the
//                                                              shifted-data form, see the kernel)
// and writes  out = act( (y - mu) * rsqrt(var + eps) * gamma + beta
//                        [ + (yp - mu_p) * rsqrt(var_p + eps) * gamma_p + beta_p ]   (projection shortcut)
//                        [ + res ] )                                                  (identity shortcut)
// act = ReLU or identity.  out may alias y (each element is read and written by the same
// thread, after the statistics).
//
// Layout: NHWC, dense; a CTA owns gpc whole groups of one image (gpc*cpg contiguous
// channels per pixel) and reads them as 16-byte vectors: thread t always handles the
// same vector slot v = t % V of the pixel row, pixels t / V, t / V + k, ... (k = threads / V),
// so its partial sums belong to one group; the partials are reduced in a fixed order
// (warp butterflies + a per-warp sum, see group_sums): deterministic and independent of B.
// HBM-bound: y is read once (held in registers, kGnPPT pixels x 16 B per thread), the shortcut
// once, out written once.
#include "slim_internal.h"

#include <cuda_bf16.h>

namespace slim {
namespace {

// 16-byte vectors are kept packed in registers (uint4: 8 bf16 or 4 fp32) and unpacked on use
template <typename T>
__device__ __forceinline__ uint4 ld16(const T *p) { return *reinterpret_cast<const uint4 *>(p); }
__device__ __forceinline__ void unpack(const uint4 &q, uint16_t, float *v) {
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        v[2 * i] = __uint_as_float(w[i] << 16);
        v[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
}
__device__ __forceinline__ void unpack(const uint4 &q, float, float *v) {
    v[0] = __uint_as_float(q.x);
    v[1] = __uint_as_float(q.y);
    v[2] = __uint_as_float(q.z);
    v[3] = __uint_as_float(q.w);
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);   // RNE
    return *reinterpret_cast<const uint32_t *>(&h);
}
__device__ __forceinline__ void store_vec(uint16_t *p, const float *v) {
    *reinterpret_cast<uint4 *>(p) = make_uint4(pack2(v[0], v[1]), pack2(v[2], v[3]), pack2(v[4], v[5]), pack2(v[6], v[7]));
}
__device__ __forceinline__ void store_vec(float *p, const float *v) {
    *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
}

constexpr int kGnMaxThreads = 512;
constexpr int kGnPPT = 8;       // pixels per thread: the CTA's slice lives in registers (y read once)
constexpr int kGnMaxCh = 512;   // channels per CTA slice

// Per-(local group) totals of one partial pair per thread, in a fixed order (deterministic,
// independent of B).  Thread t holds vector slot v = t % V (group v / vpg) of pixel lane t / V.
// Fast path (V < 32, whole warps): butterfly over the group's vpg slots and over the warp's
// pixel lanes (offsets V .. 16), one partial per (warp, group) in smem, summed over warps.
// Otherwise every thread's partial goes to smem and thread g sums its group's k*vpg partials.
__device__ __forceinline__ void group_sums(float x0, float x1, int V, int vpg, int k, int gpc, float2 *part,
                                           float *out0, float *out1) {
    const int t = threadIdx.x, lane = t & 31, nw = blockDim.x >> 5;
    if (V < 32 && (blockDim.x & 31) == 0) {
        for (int o = 1; o < vpg; o <<= 1) {
            x0 += __shfl_xor_sync(0xffffffffu, x0, o);
            x1 += __shfl_xor_sync(0xffffffffu, x1, o);
        }
        for (int o = V; o < 32; o <<= 1) {
            x0 += __shfl_xor_sync(0xffffffffu, x0, o);
            x1 += __shfl_xor_sync(0xffffffffu, x1, o);
        }
        if (lane < V && lane % vpg == 0) part[(t >> 5) * gpc + lane / vpg] = make_float2(x0, x1);
        __syncthreads();
        if (t < gpc) {
            float2 s = make_float2(0.f, 0.f);
            for (int w = 0; w < nw; ++w) {
                s.x += part[w * gpc + t].x;
                s.y += part[w * gpc + t].y;
            }
            out0[t] = s.x;
            out1[t] = s.y;
        }
    } else {
        part[t] = make_float2(x0, x1);
        __syncthreads();
        if (t < gpc) {
            float2 s = make_float2(0.f, 0.f);
            for (int m = 0; m < k; ++m)
                for (int j = 0; j < vpg; ++j) {
                    s.x += part[m * V + t * vpg + j].x;
                    s.y += part[m * V + t * vpg + j].y;
                }
            out0[t] = s.x;
            out1[t] = s.y;
        }
    }
    __syncthreads();
}

// Threads per CTA: bf16 <= 256 (3 CTAs per SM resident), fp32 <= 512 (its vectors hold 4 values).
template <typename T>
constexpr int gn_max_threads() { return sizeof(T) == 2 ? 256 : kGnMaxThreads; }

// TWO: a second raw input (the projection shortcut) -- a template flag so the common case
// keeps half the registers (more CTAs resident: the kernel is a short latency chain).
template <typename T, bool TWO>
__global__ void __launch_bounds__(gn_max_threads<T>(), sizeof(T) == 2 ? (TWO ? 2 : 4) : 1) gn_kernel(const GnArgs a) {
    constexpr int VE = 16 / sizeof(T);   // elements per 16-byte vector
    __shared__ float2 part[kGnMaxThreads];
    __shared__ float gsum[2][kGnMaxCh / 8];
    __shared__ float stat[2][2][kGnMaxCh / 8];          // [y|yp][mean|rstd][local group]
    __shared__ float coef[2][2][kGnMaxCh];              // [y|yp][A|Bc] per channel of the slice
    const int V = a.gpc * a.cpg / VE, vpg = a.cpg / VE;
    const int t = threadIdx.x, v = t % V, k = blockDim.x / V;
    constexpr bool two = TWO;
    const float inv_cnt = 1.f / (static_cast<float>(a.HW) * a.cpg);
    const int p0 = t / V;
    const int slices = a.C / (a.gpc * a.cpg);

    // programmatic dependent launch: the index math above overlaps the producing conv's tail;
    // dependents may start their prologue now (their own wait covers this grid's completion)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    // persistent over (image, slice) items: the grid may be capped (SM share of this width)
    for (int item = blockIdx.x; item < a.B * slices; item += gridDim.x) {
    const int n = item / slices;
    const int ch0 = (item - n * slices) * a.gpc * a.cpg;   // first channel of this CTA's slice
    const size_t img = static_cast<size_t>(n) * a.HW * a.C;
    const size_t base = img + ch0 + v * VE;

    // the slice into registers: pixels p0, p0 + k, ... (< kGnPPT of them), all loads in flight
    uint4 q0[kGnPPT], q1[TWO ? kGnPPT : 1];
#pragma unroll
    for (int j = 0; j < kGnPPT; ++j) {
        const int p = p0 + j * k;
        q0[j] = make_uint4(0u, 0u, 0u, 0u);
        if (TWO) q1[TWO ? j : 0] = make_uint4(0u, 0u, 0u, 0u);
        if (p < a.HW) {
            q0[j] = ld16(static_cast<const T *>(a.y) + base + static_cast<size_t>(p) * a.C);
            if (TWO) q1[TWO ? j : 0] = ld16(static_cast<const T *>(a.yp) + base + static_cast<size_t>(p) * a.C);
        }
    }
    // statistics in ONE register pass, shifted by a sample of the group (the group's first value
    // in this image, K): mean = K + S1/N, var = S2/N - (S1/N)^2 with S1 = sum(x - K),
    // S2 = sum((x - K)^2) -- K lies within a few sigma of the mean, so the subtraction does not
    // cancel (the shifted-data form of the textbook variance).  Fixed-order reductions.
    const int lg = v / vpg;
    const size_t gfirst = img + ch0 + static_cast<size_t>(lg) * a.cpg;   // pixel 0, first channel of the group
    float K0, K1 = 0.f;
    {
        float kv[VE];
        unpack(ld16(static_cast<const T *>(a.y) + gfirst), T(), kv);
        K0 = kv[0];
        if (TWO) {
            unpack(ld16(static_cast<const T *>(a.yp) + gfirst), T(), kv);
            K1 = kv[0];
        }
    }
    float s0 = 0.f, q0s = 0.f, s1 = 0.f, q1s = 0.f;
#pragma unroll
    for (int j = 0; j < kGnPPT; ++j)
        if (p0 + j * k < a.HW) {
            float x0[VE], x1[VE];
            unpack(q0[j], T(), x0);
            if (TWO) unpack(q1[TWO ? j : 0], T(), x1);
#pragma unroll
            for (int i = 0; i < VE; ++i) {
                const float d0 = x0[i] - K0;
                s0 += d0;
                q0s = fmaf(d0, d0, q0s);
                if (TWO) {
                    const float d1 = x1[i] - K1;
                    s1 += d1;
                    q1s = fmaf(d1, d1, q1s);
                }
            }
        }
    group_sums(s0, q0s, V, vpg, k, a.gpc, part, gsum[0], gsum[1]);
    if (t < a.gpc) {   // K of local group t: its first value (every thread of group t loaded the same one)
        float kv[VE];
        unpack(ld16(static_cast<const T *>(a.y) + img + ch0 + static_cast<size_t>(t) * a.cpg), T(), kv);
        const float m = gsum[0][t] * inv_cnt;
        stat[0][0][t] = kv[0] + m;
        stat[0][1][t] = rsqrtf(fmaxf(fmaf(-m, m, gsum[1][t] * inv_cnt), 0.f) + a.eps);
    }
    if (TWO) {
        __syncthreads();   // gsum is reused
        group_sums(s1, q1s, V, vpg, k, a.gpc, part, gsum[0], gsum[1]);
        if (t < a.gpc) {
            float kv[VE];
            unpack(ld16(static_cast<const T *>(a.yp) + img + ch0 + static_cast<size_t>(t) * a.cpg), T(), kv);
            const float m = gsum[0][t] * inv_cnt;
            stat[1][0][t] = kv[0] + m;
            stat[1][1][t] = rsqrtf(fmaxf(fmaf(-m, m, gsum[1][t] * inv_cnt), 0.f) + a.eps);
        }
    }
    __syncthreads();
    // per-channel affine of the slice in smem: z = y * A + Bc, A = rstd*gamma, Bc = beta - mu*A
    for (int c = t; c < a.gpc * a.cpg; c += blockDim.x) {
        const int g = c / a.cpg;
        const float A = stat[0][1][g] * a.gamma[ch0 + c];
        coef[0][0][c] = A;
        coef[0][1][c] = fmaf(-stat[0][0][g], A, a.beta[ch0 + c]);
        if (two) {
            const float Ap = stat[1][1][g] * a.gamma_p[ch0 + c];
            coef[1][0][c] = Ap;
            coef[1][1][c] = fmaf(-stat[1][0][g], Ap, a.beta_p[ch0 + c]);
        }
    }
    __syncthreads();
    const float *A0 = coef[0][0] + v * VE, *B0 = coef[0][1] + v * VE, *A1 = coef[1][0] + v * VE,
                *B1 = coef[1][1] + v * VE;
    // pass 3: apply (+ shortcut) (+ ReLU); out may alias y (every y element is already in registers).
    // pool_out (the network's last GN): the average pool of the result instead of its store --
    // per-thread channel sums, then a fixed-order sum over the k pixel lanes (deterministic)
    float zs[VE];
#pragma unroll
    for (int i = 0; i < VE; ++i) zs[i] = 0.f;
#pragma unroll
    for (int j = 0; j < kGnPPT; ++j) {
        const int p = p0 + j * k;
        if (p >= a.HW) continue;
        float z[VE], x0[VE], x1[VE], r[VE];
        unpack(q0[j], T(), x0);
        if (TWO) unpack(q1[TWO ? j : 0], T(), x1);
        unpack(a.res ? ld16(static_cast<const T *>(a.res) + base + static_cast<size_t>(p) * a.C) : make_uint4(0u, 0u, 0u, 0u),
               T(), r);
#pragma unroll
        for (int i = 0; i < VE; ++i) {
            z[i] = fmaf(x0[i], A0[i], B0[i]);
            if (two) z[i] += fmaf(x1[i], A1[i], B1[i]);
            if (a.res) z[i] += r[i];
            z[i] = fmaxf(z[i], a.relu_lo);
            zs[i] += z[i];
        }
        if (!a.pool_out) store_vec(static_cast<T *>(a.out) + base + static_cast<size_t>(p) * a.C, z);
    }
    if (a.pool_out) {
        float *red = &coef[0][0][0];   // blockDim * VE <= 2048 floats = the coef array (all reads done below)
        __syncthreads();
#pragma unroll
        for (int i = 0; i < VE; ++i) red[t * VE + i] = zs[i];
        __syncthreads();
        for (int cl = t; cl < V * VE; cl += blockDim.x) {   // local channel cl = slot * VE + element
            const int slot = cl / VE, e = cl - slot * VE;
            float sum = 0.f;
            for (int m = 0; m < k; ++m) sum += red[(m * V + slot) * VE + e];
            a.pool_out[static_cast<size_t>(n) * a.C + ch0 + cl] = sum / static_cast<float>(a.HW);
        }
        __syncthreads();   // red (= coef) is rewritten by the next item
    }
    }   // items
}

// GN apply from the producing conv's statistics partials (kernels_halo.cu, HaloArgs::gn_part): each thread
// takes 8 channels (one 16-B vector, half of a 16-channel group) of one pixel; it merges the image's
// per-tile partials of its group (Chan's pairwise update, fixed tile order -> deterministic, the same
// for every pixel of the image), then out = act(y*A + Bc [+ res]) with A = rstd*gamma, Bc = beta - mean*A.
// pool_out: per (image, 8 channels) the average over the image's pixels instead of the store.
// The coefficients of a whole image (C channels) are built once per CTA in smem: thread c merges the
// image's tiles_per_img partials of channel c's group (Chan's pairwise update, fixed tile order: the same
// for every pixel) -> A = rstd*gamma, Bc = beta - mean*A.
constexpr int kGnpThreads = 256;
constexpr int kGnpMaxC = 512;
__device__ __forceinline__ void gn_part_image_coef(const GnPartArgs &a, int n, float *sA, float *sB) {
    const int G = a.C / 16;
    for (int c = threadIdx.x; c < a.C; c += blockDim.x) {
        const float2 *p = a.part + static_cast<size_t>(n) * a.tiles_per_img * G + c / 16;
        float mean = p[0].x, m2 = p[0].y, cnt = a.part_count;
        for (int t = 1; t < a.tiles_per_img; ++t) {
            const float2 q = p[static_cast<size_t>(t) * G];
            const float nb = a.part_count, tot = cnt + nb;
            const float d = q.x - mean;
            mean = fmaf(d, nb / tot, mean);
            m2 = (m2 + q.y) + d * d * (cnt * nb / tot);
            cnt = tot;
        }
        const float rstd = rsqrtf(fmaxf(m2 / cnt, 0.f) + a.eps);
        const float A = rstd * a.gamma[c];
        sA[c] = A;
        sB[c] = fmaf(-mean, A, a.beta[c]);
    }
}

// grid: (pixel chunks of one image) x images; pool_out: one CTA per image
__global__ void __launch_bounds__(kGnpThreads) gn_apply_part_kernel(const GnPartArgs a, int px_per_cta) {
    __shared__ float sA[kGnpMaxC], sB[kGnpMaxC];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int V = a.C / 8;
    const int chunks = a.pool_out ? 1 : (a.HW + px_per_cta - 1) / px_per_cta;
    for (int item = blockIdx.x; item < a.B * chunks; item += gridDim.x) {
        const int n = item / chunks, ck = item - n * chunks;
        __syncthreads();   // the previous item's readers of sA / sB are done
        gn_part_image_coef(a, n, sA, sB);
        __syncthreads();
        if (a.pool_out) {   // thread per 8 channels: the image's pixels summed in order, then / HW
            for (int v = threadIdx.x; v < V; v += blockDim.x) {
                const int c8 = v * 8;
                float acc[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) acc[k] = 0.f;
                for (int p = 0; p < a.HW; ++p) {
                    const size_t o = (static_cast<size_t>(n) * a.HW + p) * a.C + c8;
                    float y[8], r[8];
                    unpack(ld16(a.y + o), uint16_t(), y);
                    unpack(a.res ? ld16(a.res + o) : make_uint4(0u, 0u, 0u, 0u), uint16_t(), r);
#pragma unroll
                    for (int k = 0; k < 8; ++k) acc[k] += fmaxf(fmaf(y[k], sA[c8 + k], sB[c8 + k]) + r[k], a.relu_lo);
                }
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    a.pool_out[static_cast<size_t>(n) * a.C + c8 + k] = acc[k] / static_cast<float>(a.HW);
            }
            continue;
        }
        const int p0 = ck * px_per_cta, p1 = min(a.HW, p0 + px_per_cta);
        const long lo = static_cast<long>(p0) * V, hi = static_cast<long>(p1) * V;
        const size_t img = static_cast<size_t>(n) * a.HW * a.C;
        for (long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
            const int c8 = static_cast<int>(i % V) * 8;
            const size_t o = img + static_cast<size_t>(i) * 8;
            float y[8], r[8], z[8];
            unpack(ld16(a.y + o), uint16_t(), y);
            unpack(a.res ? ld16(a.res + o) : make_uint4(0u, 0u, 0u, 0u), uint16_t(), r);
#pragma unroll
            for (int k = 0; k < 8; ++k) z[k] = fmaxf(fmaf(y[k], sA[c8 + k], sB[c8 + k]) + r[k], a.relu_lo);
            store_vec(a.out + o, z);
        }
    }
}

}  // namespace

cudaError_t launch_gn_apply_part(const GnPartArgs &a, cudaStream_t s, bool pdl) {
    if (a.C % 16 || a.C > kGnpMaxC || a.B < 1 || a.HW < 1 || a.tiles_per_img < 1) return cudaErrorInvalidValue;
    // pixel chunk per CTA: about 2048 16-B vectors (8 per thread)
    int px = 2048 / (a.C / 8);
    if (px < 1) px = 1;
    if (px > a.HW) px = a.HW;
    const long items = a.pool_out ? a.B : static_cast<long>(a.B) * ((a.HW + px - 1) / px);
    const long cap = a.max_ctas > 0 ? a.max_ctas : 148L * 8;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(items < cap ? items : cap));
    cfg.blockDim = dim3(kGnpThreads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, gn_apply_part_kernel, a, px);
}

// Pixel lanes per vector slot: k = HW / kGnPPT (each thread holds kGnPPT pixels).
static int gn_lanes(int HW) { return HW > kGnPPT ? (HW + kGnPPT - 1) / kGnPPT : 1; }

int gn_groups_per_cta(int /*B*/, int HW, int C, int cpg, bool fp32) {
    // independent of B (batch independence is bit-exact): widen the slice while it divides
    // G and the CTA stays within its thread budget (vpg = cpg/8 vectors per group in bf16, cpg/4 in fp32)
    const int G = C / cpg, k = gn_lanes(HW), vpg = cpg / (fp32 ? 4 : 8);
    const int maxt = fp32 ? gn_max_threads<float>() : gn_max_threads<uint16_t>();
    int gpc = 1;
    while (G % (2 * gpc) == 0 && 2 * gpc * vpg * k <= maxt && 2 * gpc * cpg <= kGnMaxCh) gpc *= 2;
    return gpc;
}

cudaError_t launch_gn(const GnArgs &a, bool fp32, cudaStream_t s, bool pdl) {
    const int VE = fp32 ? 4 : 8;
    if (a.cpg % VE || a.C % (a.gpc * a.cpg) || a.gpc * a.cpg > kGnMaxCh || a.HW < 1) return cudaErrorInvalidValue;
    const int V = a.gpc * a.cpg / VE;
    int k = 1;   // power-of-two pixel lanes per vector slot, every thread holds <= kGnPPT pixels
    while (k < gn_lanes(a.HW)) k *= 2;
    if (V * k > (fp32 ? gn_max_threads<float>() : gn_max_threads<uint16_t>()) || (a.HW + k - 1) / k > kGnPPT)
        return cudaErrorInvalidValue;
    cudaLaunchConfig_t cfg{};
    const int items = a.B * (a.C / (a.gpc * a.cpg));
    cfg.gridDim = dim3(a.max_ctas > 0 && a.max_ctas < items ? a.max_ctas : items);
    cfg.blockDim = dim3(V * k);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    if (a.yp)
        return fp32 ? cudaLaunchKernelEx(&cfg, gn_kernel<float, true>, a) : cudaLaunchKernelEx(&cfg, gn_kernel<uint16_t, true>, a);
    return fp32 ? cudaLaunchKernelEx(&cfg, gn_kernel<float, false>, a) : cudaLaunchKernelEx(&cfg, gn_kernel<uint16_t, false>, a);
}

}  // namespace slim
