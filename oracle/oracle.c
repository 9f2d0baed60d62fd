/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.  The plain, slow, obviously correct CPU
 * definition of the width-sliced convolution on the Slim Scheduler hot path.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library.  It shares no code, header, table or
 * constant with the CUDA path (paper_2510_09018_b200/csrc) and includes nothing
 * from it.
 *
 * Arithmetic: IEEE fp64 throughout (task rule: fp64 unless the paper fixes the
 * precision; PAPER.md never states one).  Summation order is fixed: kh, kw, ci
 * ascending, exactly as the definition is written below.
 *
 * What it computes (PyTorch cross-correlation semantics):
 *
 *   y[n,oh,ow,co] = sum_{kh<k} sum_{kw<k} sum_{ci<c_in}
 *                     x[n, s*oh+kh-p, s*ow+kw-p, ci] * w[co,kh,kw,ci]
 *
 * with out-of-range input terms omitted (zero padding),
 * H_o = floor((H_i + 2p - k)/s) + 1, and only co < c_out, ci < c_in of the
 * FULL-width shared weight tensor w[Cout_full][k][k][Cin_full] read -- the
 * "universal width slicing" of PAPER.md:49 ("segmented, universally slimmable
 * backbone") / PAPER.md:148 ("Each segment supports width ratios w") as stated
 * by the north_star ("first ceil(r*C) input/output channels of shared weights").
 *
 * Parallelism: OpenMP over (n, oh) rows only; each output element is still the
 * single sequential sum above, so results do not depend on the thread count.
 *
 * Two entry points compute the SAME definition with the SAME per-output summation
 * order (kh, kw, ci ascending, one rounded multiply and one rounded add per term,
 * no FMA contraction: -ffp-contract=off):
 *   oracle_conv2d_plain : the loop nest exactly as the formula reads (one output
 *                         element at a time) -- the reference for the one below;
 *   oracle_conv2d       : the loops over (kh, kw, ci) moved outside the loop over co,
 *                         so the c_out independent sums of one output pixel advance
 *                         together and the compiler can vectorise ACROSS outputs (no
 *                         reassociation inside any one sum).  Bitwise identical to
 *                         the plain form (tests/test_oracle_pins.py pins this); it
 *                         only makes the >= 4096-image argmax checks affordable.
 */
#include <omp.h>
#include <stddef.h>
#include <stdlib.h>

int oracle_version(void) { return 2; }

/* Thread count of the OpenMP loops (bench.py's cpu_baseline times 1 thread and all threads). */
void oracle_set_num_threads(int n) { omp_set_num_threads(n > 0 ? n : 1); }
int oracle_max_threads(void) { return omp_get_max_threads(); }

/* Output spatial size of a k x k, stride s, padding p convolution (O2). */
long oracle_out_size(long h_in, long k, long s, long p) { return (h_in + 2 * p - k) / s + 1; }

/*
 * x : dense activations [B][H][W][c_in]           (NHWC, c_in = active input channels)
 * w : full-width weights [cout_full][k][k][cin_full] (KRSC); entries with
 *     co >= c_out or ci >= c_in are never read (they may hold NaN).
 * y : dense output [B][Ho][Wo][c_out]
 * Returns 0, or -1 on an argument error (nothing written).
 */
int oracle_conv2d_plain(const double *x, long B, long H, long W, long c_in,
                  const double *w, long cout_full, long k, long cin_full, long c_out,
                  long s, long p, double *y)
{
    if (B < 0 || H < 1 || W < 1 || c_in < 1 || c_in > cin_full || c_out < 1 || c_out > cout_full ||
        k < 1 || s < 1 || p < 0)
        return -1;
    const long Ho = oracle_out_size(H, k, s, p);
    const long Wo = oracle_out_size(W, k, s, p);
    if (Ho < 1 || Wo < 1) return -1;

    long row;
#pragma omp parallel for schedule(static)
    for (row = 0; row < B * Ho; ++row) {
        const long n = row / Ho, oh = row % Ho;
        for (long ow = 0; ow < Wo; ++ow) {
            double *yo = y + ((n * Ho + oh) * Wo + ow) * c_out;
            for (long co = 0; co < c_out; ++co) {
                double acc = 0.0;
                for (long kh = 0; kh < k; ++kh) {
                    const long ih = s * oh + kh - p;
                    if (ih < 0 || ih >= H) continue;          /* zero padding: term omitted */
                    for (long kw = 0; kw < k; ++kw) {
                        const long iw = s * ow + kw - p;
                        if (iw < 0 || iw >= W) continue;
                        const double *xi = x + ((n * H + ih) * W + iw) * c_in;
                        const double *wi = w + ((co * k + kh) * k + kw) * cin_full;
                        for (long ci = 0; ci < c_in; ++ci) acc += xi[ci] * wi[ci];
                    }
                }
                yo[co] = acc;
            }
        }
    }
    return 0;
}

/*
 * Same arguments, same result (bitwise) as oracle_conv2d_plain.
 *
 * Layout only (no arithmetic): the active weight slice w[:c_out, :, :, :c_in] is copied
 * to wt[kh][kw][ci][co], and x to a zero-padded copy xp[n][H+2p][W+2p][c_in], so every
 * tap of every output lands inside xp.  A tap that falls in the padding then contributes
 * the product 0 * w = +-0 instead of being omitted; that leaves the running sum unchanged
 * bit for bit (the sum starts at +0 and, in round-to-nearest, a sum is -0 only when both
 * addends are -0, so it is never -0; acc + (+-0) == acc for acc != 0 and +0 + (+-0) == +0),
 * for the finite weights of the active slice.  Each output's terms are still added one
 * at a time in kh, kw, ci order; only independent outputs are interleaved: blocks of
 * 4 pixels x 16 output channels advance together (vectorised across co), the generic
 * path (any c_out, any Wo) one pixel x all channels at a time.
 */
#if defined(__GNUC__) && !defined(__clang__) && defined(__x86_64__)
#define ORACLE_CLONES __attribute__((target_clones("avx512f", "avx2", "default")))
#else
#define ORACLE_CLONES
#endif

typedef double v8d __attribute__((vector_size(64)));   /* GCC vector extension: 8 lanes */

/* Blocked path (c_out % 16 == 0, Wo % 4 == 0): wb[cc][kh][kw][ci][16] holds output channels
 * 16cc..16cc+15, so one chunk's weights stay cache-resident while it sweeps every row. */
ORACLE_CLONES
static void conv_blocked(const double *restrict xp, long B, long Hp, long Wp, long c_in,
                         const double *restrict wb, long k, long c_out, long s, long Ho, long Wo,
                         double *restrict y)
{
    const long rows = B * Ho, nchunk = c_out / 16, xs = s * c_in;
    long t;
#pragma omp parallel for schedule(static)
    for (t = 0; t < nchunk * rows; ++t) {
        const long cc = t / rows, row = t % rows;
        const long n = row / Ho, oh = row % Ho;
        const double *restrict wc = wb + cc * k * k * c_in * 16;
        for (long ow0 = 0; ow0 < Wo; ow0 += 4) {
            /* 4 pixels x 16 channels of independent sums, held as 8 vectors of 8 */
            v8d a0 = {0}, a1 = {0}, a2 = {0}, a3 = {0}, b0 = {0}, b1 = {0}, b2 = {0}, b3 = {0};
            for (long kh = 0; kh < k; ++kh) {
                for (long kw = 0; kw < k; ++kw) {
                    const double *restrict xr = xp + ((n * Hp + s * oh + kh) * Wp + s * ow0 + kw) * c_in;
                    const double *restrict wk = wc + (kh * k + kw) * c_in * 16;
                    for (long ci = 0; ci < c_in; ++ci) {
                        v8d wlo, whi;
                        __builtin_memcpy(&wlo, wk + ci * 16, sizeof wlo);
                        __builtin_memcpy(&whi, wk + ci * 16 + 8, sizeof whi);
                        const double x0 = xr[ci], x1 = xr[xs + ci], x2 = xr[2 * xs + ci], x3 = xr[3 * xs + ci];
                        a0 += x0 * wlo; b0 += x0 * whi;
                        a1 += x1 * wlo; b1 += x1 * whi;
                        a2 += x2 * wlo; b2 += x2 * whi;
                        a3 += x3 * wlo; b3 += x3 * whi;
                    }
                }
            }
            double *restrict o = y + ((n * Ho + oh) * Wo + ow0) * c_out + cc * 16;
            __builtin_memcpy(o, &a0, sizeof a0);               __builtin_memcpy(o + 8, &b0, sizeof b0);
            __builtin_memcpy(o + c_out, &a1, sizeof a1);       __builtin_memcpy(o + c_out + 8, &b1, sizeof b1);
            __builtin_memcpy(o + 2 * c_out, &a2, sizeof a2);   __builtin_memcpy(o + 2 * c_out + 8, &b2, sizeof b2);
            __builtin_memcpy(o + 3 * c_out, &a3, sizeof a3);   __builtin_memcpy(o + 3 * c_out + 8, &b3, sizeof b3);
        }
    }
}

/* Generic path: one pixel x all c_out channels at a time; wt[kh][kw][ci][co]. */
ORACLE_CLONES
static void conv_rows(const double *restrict xp, long B, long Hp, long Wp, long c_in,
                      const double *restrict wt, long k, long c_out, long s, long Ho, long Wo,
                      double *restrict y)
{
    long row;
#pragma omp parallel for schedule(static)
    for (row = 0; row < B * Ho; ++row) {
        const long n = row / Ho, oh = row % Ho;
        for (long ow = 0; ow < Wo; ++ow) {
            double *restrict acc = y + ((n * Ho + oh) * Wo + ow) * c_out;
            for (long co = 0; co < c_out; ++co) acc[co] = 0.0;
            for (long kh = 0; kh < k; ++kh) {
                for (long kw = 0; kw < k; ++kw) {
                    const double *restrict xi = xp + ((n * Hp + s * oh + kh) * Wp + s * ow + kw) * c_in;
                    const double *restrict wk = wt + (kh * k + kw) * c_in * c_out;
                    for (long ci = 0; ci < c_in; ++ci) {
                        const double xv = xi[ci];
                        const double *restrict wc = wk + ci * c_out;
                        for (long co = 0; co < c_out; ++co) acc[co] += xv * wc[co];
                    }
                }
            }
        }
    }
}

int oracle_conv2d(const double *x, long B, long H, long W, long c_in,
                  const double *w, long cout_full, long k, long cin_full, long c_out,
                  long s, long p, double *y)
{
    if (B < 0 || H < 1 || W < 1 || c_in < 1 || c_in > cin_full || c_out < 1 || c_out > cout_full ||
        k < 1 || s < 1 || p < 0)
        return -1;
    const long Ho = oracle_out_size(H, k, s, p);
    const long Wo = oracle_out_size(W, k, s, p);
    if (Ho < 1 || Wo < 1) return -1;
    if (B == 0) return 0;
    /* padded extent: every tap s*o + kh of every output lies inside [0, Hp) */
    const long Hp = (Ho - 1) * s + k > H + 2 * p ? (Ho - 1) * s + k : H + 2 * p;
    const long Wp = (Wo - 1) * s + k > W + 2 * p ? (Wo - 1) * s + k : W + 2 * p;
    double *wt = (double *)malloc(sizeof(double) * (size_t)(k * k * c_in * c_out));
    double *xp = (double *)calloc((size_t)(B * Hp * Wp * c_in), sizeof(double));
    if (!wt || !xp) { free(wt); free(xp); return -1; }
    const int blocked = (c_out % 16 == 0) && (Wo % 4 == 0);
    for (long co = 0; co < c_out; ++co)
        for (long kh = 0; kh < k; ++kh)
            for (long kw = 0; kw < k; ++kw)
                for (long ci = 0; ci < c_in; ++ci) {
                    const double v = w[((co * k + kh) * k + kw) * cin_full + ci];
                    if (blocked)
                        wt[((((co / 16) * k + kh) * k + kw) * c_in + ci) * 16 + co % 16] = v;
                    else
                        wt[((kh * k + kw) * c_in + ci) * c_out + co] = v;
                }
    for (long n = 0; n < B; ++n)
        for (long ih = 0; ih < H; ++ih)
            for (long iw = 0; iw < W; ++iw)
                for (long ci = 0; ci < c_in; ++ci)
                    xp[((n * Hp + ih + p) * Wp + iw + p) * c_in + ci] = x[((n * H + ih) * W + iw) * c_in + ci];
    if (blocked)
        conv_blocked(xp, B, Hp, Wp, c_in, wt, k, c_out, s, Ho, Wo, y);
    else
        conv_rows(xp, B, Hp, Wp, c_in, wt, k, c_out, s, Ho, Wo, y);
    free(wt);
    free(xp);
    return 0;
}
