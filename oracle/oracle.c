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
 */
#include <stddef.h>

int oracle_version(void) { return 1; }

/* Output spatial size of a k x k, stride s, padding p convolution (O2). */
long oracle_out_size(long h_in, long k, long s, long p) { return (h_in + 2 * p - k) / s + 1; }

/*
 * x : dense activations [B][H][W][c_in]           (NHWC, c_in = active input channels)
 * w : full-width weights [cout_full][k][k][cin_full] (KRSC); entries with
 *     co >= c_out or ci >= c_in are never read (they may hold NaN).
 * y : dense output [B][Ho][Wo][c_out]
 * Returns 0, or -1 on an argument error (nothing written).
 */
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
