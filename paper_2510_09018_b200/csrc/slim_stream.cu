// slim_stream.cu -- native request-stream executor (CFG4; PAPER.md P:49 key re-entry, Alg. 1
// l.3-4 batch formation + l.10 RUNBATCH; include/slim.h "native request-stream executor").
//
// The Python StreamExecutor (stream.py) spends ~10 us of interpreter time per packed batch on
// marshalling; a fresh routed stream (new batch shapes every step, so no graph replay) then runs
// host-bound.  This is the same sequencing in C++: per call
//
//   pack all four segments on the host (slim_pack; keys depend only on the tuples)
//   one H2D copy of the four request orders (double-buffered pinned staging)
//   for s in 0..3:  [fork lanes]  for each batch: slim_launch (gather + segment), slim_scatter  [join]
//
// Data layout: pools[s] (s = 1..3) hold one row per request, sized for the widest previous width
// (h*h*act_channels(w_max, C_{s-1}) elements, dense prefix = the request's own width); segment 0
// gathers straight from the caller's images.  Each lane owns a slab (gathered batch), an out
// buffer (the batch's outputs before the scatter) and a forward workspace, all sized for B_max.
#include <chrono>
#include <cmath>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/slim.h"

namespace slim {
const slim_config *ctx_config(const slim_ctx *ctx);   // slim_api.cu
}

struct slim_stream {
    slim_ctx *ctx = nullptr;
    slim_config cfg{};
    int n_max = 0, B_max = 0, lanes = 1, nw = 0;
    size_t eb = 2, row_bytes[4] = {}, out_bytes = 0, wsb = 0;
    void *pools[4] = {};
    std::vector<void *> slab, out, ws;
    std::vector<cudaStream_t> lane_stream;     // lanes > 1 only
    std::vector<cudaEvent_t> lane_done;        // join events, one per lane
    cudaEvent_t fork = nullptr;
    uint32_t *order_h[2] = {};                 // pinned staging, used alternately
    cudaEvent_t order_ev[2] = {};              // the H2D copy that last read order_h[i]
    bool order_ev_live[2] = {};
    int buf = 0;
    uint32_t *order_d = nullptr;               // device: 4 * n_max request indices
    std::vector<slim_request> q;
    std::vector<slim_launch_desc> descs[4];
    int n_descs[4] = {};
};

namespace {

int width_slot(const slim_config &c, float r) {   // same matching as slim_pack's key validation
    for (int i = 0; i < c.n_widths; ++i)
        if (std::fabs(c.widths[i] - r) < 1e-6f) return i;
    return 0;   // (unreachable: slim_pack rejected the stream)
}

}  // namespace

extern "C" {

void slim_stream_destroy(slim_stream *x) {
    if (!x) return;
    cudaDeviceSynchronize();
    for (void *p : x->slab) cudaFree(p);
    for (void *p : x->out) cudaFree(p);
    for (void *p : x->ws) cudaFree(p);
    for (cudaStream_t s : x->lane_stream) cudaStreamDestroy(s);
    for (cudaEvent_t e : x->lane_done) cudaEventDestroy(e);
    if (x->fork) cudaEventDestroy(x->fork);
    for (int i = 0; i < 2; ++i) {
        if (x->order_h[i]) cudaFreeHost(x->order_h[i]);
        if (x->order_ev[i]) cudaEventDestroy(x->order_ev[i]);
    }
    cudaFree(x->order_d);
    for (int s = 1; s < 4; ++s) cudaFree(x->pools[s]);
    delete x;
}

slim_status slim_stream_create(slim_ctx *ctx, int n_max, int B_max, int lanes, slim_stream **out) {
    if (!out) return SLIM_EINVAL;
    *out = nullptr;
    if (!ctx || n_max < 1 || B_max < 1 || lanes < 1 || lanes > 16) return SLIM_EINVAL;
    const slim_config &c = *slim::ctx_config(ctx);
    if (B_max > c.max_batch) return SLIM_EINVAL;
    slim_stream *x = new slim_stream();
    x->ctx = ctx;
    x->cfg = c;
    x->n_max = n_max;
    x->B_max = B_max;
    x->lanes = lanes;
    x->nw = c.n_widths;
    x->eb = c.dtype == SLIM_BF16 ? 2 : 4;
    const float wmax = c.widths[c.n_widths - 1];
    x->row_bytes[0] = static_cast<size_t>(c.image_hw) * c.image_hw * c.in_channels * x->eb;
    size_t widest = x->row_bytes[0];
    for (int s = 1; s < 4; ++s) {
        const size_t h = static_cast<size_t>(c.image_hw >> (s - 1));
        x->row_bytes[s] = h * h * slim_act_channels(wmax, c.base_channels[s - 1]) * x->eb;
        widest = x->row_bytes[s] > widest ? x->row_bytes[s] : widest;
    }
    x->out_bytes = widest > static_cast<size_t>(c.num_classes) * 4 ? widest : static_cast<size_t>(c.num_classes) * 4;
    for (int s = 0; s < 4; ++s) {
        const size_t b = slim_forward_workspace_bytes(ctx, s, wmax, wmax, B_max);
        x->wsb = b > x->wsb ? b : x->wsb;
    }
    bool ok = true;
    for (int s = 1; s < 4 && ok; ++s)
        ok = cudaMalloc(&x->pools[s], static_cast<size_t>(n_max) * x->row_bytes[s]) == cudaSuccess;
    x->slab.assign(lanes, nullptr);
    x->out.assign(lanes, nullptr);
    x->ws.assign(lanes, nullptr);
    for (int l = 0; l < lanes && ok; ++l)
        ok = cudaMalloc(&x->slab[l], B_max * x->out_bytes) == cudaSuccess &&   // out_bytes >= every input row
             cudaMalloc(&x->out[l], B_max * x->out_bytes) == cudaSuccess &&
             cudaMalloc(&x->ws[l], x->wsb > 0 ? x->wsb : 16) == cudaSuccess;
    if (ok && lanes > 1) {
        x->lane_stream.assign(lanes, nullptr);
        x->lane_done.assign(lanes, nullptr);
        for (int l = 0; l < lanes && ok; ++l)
            ok = cudaStreamCreateWithFlags(&x->lane_stream[l], cudaStreamNonBlocking) == cudaSuccess &&
                 cudaEventCreateWithFlags(&x->lane_done[l], cudaEventDisableTiming) == cudaSuccess;
        ok = ok && cudaEventCreateWithFlags(&x->fork, cudaEventDisableTiming) == cudaSuccess;
    }
    for (int i = 0; i < 2 && ok; ++i)
        ok = cudaMallocHost(&x->order_h[i], 4 * sizeof(uint32_t) * n_max) == cudaSuccess &&
             cudaEventCreateWithFlags(&x->order_ev[i], cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaMalloc(&x->order_d, 4 * sizeof(uint32_t) * n_max) == cudaSuccess;
    if (!ok) {
        cudaGetLastError();
        slim_stream_destroy(x);
        return SLIM_ENOMEM;
    }
    x->q.resize(n_max);
    for (int s = 0; s < 4; ++s) x->descs[s].resize(n_max);
    *out = x;
    return SLIM_OK;
}

slim_status slim_stream_run(slim_stream *x, const void *images, const float *tuples, int n, float *logits,
                            void *stream, slim_stream_stats *stats) {
    if (!x || !images || !tuples || !logits || n < 1 || n > x->n_max) return SLIM_EINVAL;
    const auto t0 = std::chrono::steady_clock::now();
    const slim_config &c = x->cfg;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    // the staging buffer of this call was last read by the copy of the call before the previous one
    const int b = x->buf;
    if (x->order_ev_live[b] && cudaEventSynchronize(x->order_ev[b]) != cudaSuccess) return SLIM_ECUDA;
    uint32_t *oh = x->order_h[b];
    const auto tp = std::chrono::steady_clock::now();
    // 1. Alg. 1 l.3-4 per segment: key (s, w_s, w_{s-1}) batches, FIFO order
    for (int s = 0; s < 4; ++s) {
        for (int i = 0; i < n; ++i)
            x->q[i] = slim_request{static_cast<uint64_t>(i), s, tuples[4 * i + s], s ? tuples[4 * i + s - 1] : 0.f,
                                   static_cast<uint32_t>(i)};
        if (slim_status e = slim_pack(&c, x->q.data(), n, x->B_max, x->descs[s].data(), n, &x->n_descs[s], oh + s * n))
            return e;
    }
    const auto t1 = std::chrono::steady_clock::now();
    // 2. the four orders in one copy, ordered on the caller's stream before the lanes fork from it
    if (cudaMemcpyAsync(x->order_d, oh, 4 * sizeof(uint32_t) * n, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaEventRecord(x->order_ev[b], st) != cudaSuccess)
        return SLIM_ECUDA;
    x->order_ev_live[b] = true;
    x->buf ^= 1;
    const uint64_t l0 = slim_launch_count(x->ctx);
    int batches = 0;
    const int lanes = x->lanes, nw = x->nw;
    const int rot = lanes / nw > 1 ? lanes / nw : 1;
    int per_width[16];
    for (int s = 0; s < 4; ++s) {
        if (lanes > 1) {   // fork: every lane starts after the previous segment's scatters
            if (cudaEventRecord(x->fork, st) != cudaSuccess) return SLIM_ECUDA;
            for (int l = 0; l < lanes; ++l)
                if (cudaStreamWaitEvent(x->lane_stream[l], x->fork, 0) != cudaSuccess) return SLIM_ECUDA;
        }
        std::memset(per_width, 0, sizeof(per_width));
        const void *pool = s == 0 ? images : x->pools[s];
        for (int k = 0; k < x->n_descs[s]; ++k) {
            const slim_launch_desc &d = x->descs[s][k];
            const int wi = width_slot(c, d.r);
            const int j = per_width[wi]++;
            const int lane = (wi + nw * (j % rot)) % lanes;
            const cudaStream_t ls = lanes > 1 ? x->lane_stream[lane] : st;
            const uint32_t *idx = x->order_d + static_cast<size_t>(s) * n + d.first;
            slim_launch_desc dl = d;
            dl.first = 0;
            if (slim_status e = slim_launch(x->ctx, &dl, idx, pool, x->row_bytes[s], x->slab[lane], x->out[lane],
                                            x->ws[lane], x->wsb, ls))
                return e;
            slim_status e;
            if (s < 3) {
                const size_t h = static_cast<size_t>(c.image_hw >> s);
                const size_t row = h * h * slim_act_channels(d.r, c.base_channels[s]) * x->eb;
                e = slim_scatter(x->ctx, x->out[lane], idx, d.batch, row, x->pools[s + 1], x->row_bytes[s + 1], ls);
            } else {
                e = slim_scatter(x->ctx, x->out[lane], idx, d.batch, c.num_classes * 4, logits, c.num_classes * 4, ls);
            }
            if (e) return e;
            ++batches;
        }
        if (lanes > 1)   // join before the next segment gathers from the pools
            for (int l = 0; l < lanes; ++l)
                if (cudaEventRecord(x->lane_done[l], x->lane_stream[l]) != cudaSuccess ||
                    cudaStreamWaitEvent(st, x->lane_done[l], 0) != cudaSuccess)
                    return SLIM_ECUDA;
    }
    if (stats) {
        stats->batches = batches;
        stats->launches = static_cast<int>(slim_launch_count(x->ctx) - l0);
        stats->pack_seconds = std::chrono::duration<double>(t1 - tp).count();
        stats->host_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    return slim_last_error(x->ctx);
}

}  // extern "C"
