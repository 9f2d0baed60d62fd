// slim_exec.cu -- native Alg. 1 executor: the LOOP of
// Algorithm 1 driven in C++ on one GPU, so the per-batch host cost is a few microseconds
// instead of the Python loop's ~100 us (executor.py keeps the Python version, with offload).
//
//   repeat until every request has finished segment 3:
//     act = slim_sched_next(now, util, vram)          (l.3-9: head-key batch, best fit, CANLOAD)
//     RUN     -> slots H2D on the instance's stream, slim_launch (gather + segment kernels),
//                slim_scatter of the outputs to the next segment's pool (or the logits),
//                event record                            (l.10 RUNBATCH)
//     IDLE / REQUEUE -> poll the in-flight events; a finished batch releases its instance
//                (slim_sched_complete) and re-enqueues its requests with key
//                (s+1, w_{s+1}, w_s); then UNLOADERLOOP (l.21-25)
//
// Instance resources (stream, event, slab, out, workspace, slot buffers) are kept in a free
// list and reused: an unloaded instance returns its buffers to the list, so the loop never
// calls cudaMalloc / cudaFree (which would synchronise the device).
#include <chrono>
#include <cstring>
#include <unordered_map>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/slim.h"

namespace slim {
const slim_config *ctx_config(const slim_ctx *ctx);   // slim_api.cu
}

namespace {

struct Res {
    cudaStream_t stream = nullptr;
    cudaEvent_t event = nullptr;
    void *slab = nullptr, *out = nullptr, *ws = nullptr;
    uint32_t *slots_d = nullptr, *slots_h = nullptr;
};

struct Pending {
    int inst, seg, batch;
    Res *res;
    std::vector<uint64_t> ids;
};

}  // namespace

struct slim_exec {
    slim_ctx *ctx = nullptr;
    slim_sched *sched = nullptr;
    slim_config cfg{};
    int n_max = 0, B_max = 0;
    size_t eb = 2, row_bytes[4] = {}, out_bytes = 0, wsb = 0, pool_bytes = 0;
    void *pools[4] = {};                       // pools[1..3]: per-request input rows of segments 1..3
    std::vector<Res *> free_res;
    std::unordered_map<int, Res *> inst_res;
    std::vector<Res *> all_res;
};

namespace {

slim_status new_res(slim_exec *x, Res **out) {
    Res *r = new Res();
    x->all_res.push_back(r);
    if (cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&r->event, cudaEventDisableTiming) != cudaSuccess ||
        cudaMalloc(&r->slab, x->B_max * x->out_bytes) != cudaSuccess ||   // out_bytes >= every input row
        cudaMalloc(&r->out, x->B_max * x->out_bytes) != cudaSuccess || cudaMalloc(&r->ws, x->wsb) != cudaSuccess ||
        cudaMalloc(&r->slots_d, x->B_max * sizeof(uint32_t)) != cudaSuccess ||
        cudaMallocHost(&r->slots_h, x->B_max * sizeof(uint32_t)) != cudaSuccess) {
        cudaGetLastError();
        return SLIM_ENOMEM;
    }
    *out = r;
    return SLIM_OK;
}

}  // namespace

extern "C" {

slim_status slim_exec_create(slim_ctx *ctx, slim_sched *sched, int n_max, int B_max, slim_exec **out) {
    if (!out) return SLIM_EINVAL;
    *out = nullptr;
    if (!ctx || !sched || n_max < 1 || B_max < 1) return SLIM_EINVAL;
    slim_exec *x = new slim_exec();
    x->ctx = ctx;
    x->sched = sched;
    x->cfg = *slim::ctx_config(ctx);
    const slim_config &c = x->cfg;
    // slim_sched_next writes up to the scheduler's B_max slots/ids into buffers sized for B_max
    if (B_max > c.max_batch || slim_sched_b_max(sched) > B_max) {
        delete x;
        return SLIM_EINVAL;
    }
    x->n_max = n_max;
    x->B_max = B_max;
    x->eb = c.dtype == SLIM_BF16 ? 2 : 4;
    const float wmax = c.widths[c.n_widths - 1];
    x->row_bytes[0] = static_cast<size_t>(c.image_hw) * c.image_hw * c.in_channels * x->eb;
    size_t widest = x->row_bytes[0];
    for (int s = 1; s < 4; ++s) {
        const size_t h = static_cast<size_t>(c.image_hw >> (s - 1));
        x->row_bytes[s] = h * h * slim_act_channels(wmax, c.base_channels[s - 1]) * x->eb;
        widest = x->row_bytes[s] > widest ? x->row_bytes[s] : widest;
    }
    // segment outputs: the widest next-segment row, or the fp32 logits of segment 3
    x->out_bytes = widest > static_cast<size_t>(c.num_classes) * 4 ? widest : static_cast<size_t>(c.num_classes) * 4;
    x->wsb = 0;
    for (int s = 0; s < 4; ++s) {
        const size_t b = slim_forward_workspace_bytes(ctx, s, wmax, wmax, B_max);
        x->wsb = b > x->wsb ? b : x->wsb;
    }
    for (int s = 1; s < 4; ++s) x->pool_bytes += static_cast<size_t>(n_max) * x->row_bytes[s];
    for (int s = 1; s < 4; ++s)
        if (cudaMalloc(&x->pools[s], static_cast<size_t>(n_max) * x->row_bytes[s]) != cudaSuccess) {
            cudaGetLastError();
            slim_exec_destroy(x);
            return SLIM_ENOMEM;
        }
    *out = x;
    return SLIM_OK;
}

void slim_exec_destroy(slim_exec *x) {
    if (!x) return;
    cudaDeviceSynchronize();
    for (Res *r : x->all_res) {
        if (r->stream) cudaStreamDestroy(r->stream);
        if (r->event) cudaEventDestroy(r->event);
        cudaFree(r->slab);
        cudaFree(r->out);
        cudaFree(r->ws);
        cudaFree(r->slots_d);
        if (r->slots_h) cudaFreeHost(r->slots_h);
        delete r;
    }
    for (int s = 1; s < 4; ++s) cudaFree(x->pools[s]);
    delete x;
}

slim_status slim_exec_run(slim_exec *x, const void *images, const float *tuples, int n, float *logits,
                          size_t vram_external, slim_exec_stats *stats, void *stream, const double *arrival_s,
                          double *done_s) {
    if (!x || !images || !tuples || !logits || n < 1 || n > x->n_max) return SLIM_EINVAL;
    if (arrival_s)
        for (int i = 1; i < n; ++i)
            if (arrival_s[i] < arrival_s[i - 1]) return SLIM_EINVAL;   // arrivals in request order
    const slim_config &c = x->cfg;
    slim_exec_stats st{};
    // the inputs are ordered before the instance streams read them
    if (cudaStreamSynchronize(static_cast<cudaStream_t>(stream)) != cudaSuccess) return SLIM_ECUDA;
    const auto t0 = std::chrono::steady_clock::now();
    auto now = [&]() { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
    // open loop: request i enters Q (key (0, w_0)) once now >= arrival_s[i]; closed loop: all at t = 0
    int admitted = 0;
    std::vector<slim_request> arrive;
    auto admit = [&](double t) -> slim_status {
        arrive.clear();
        while (admitted < n && (!arrival_s || arrival_s[admitted] <= t)) {
            const int i = admitted++;
            arrive.push_back(slim_request{static_cast<uint64_t>(i), 0, tuples[4 * i], 0.f, static_cast<uint32_t>(i)});
        }
        return arrive.empty() ? SLIM_OK : slim_sched_enqueue(x->sched, arrive.data(), static_cast<int>(arrive.size()), t);
    };
    auto arrival_due = [&]() { return admitted < n && arrival_s[admitted] <= now(); };
    std::vector<Pending> pending;
    std::vector<uint32_t> slots(x->B_max);
    std::vector<uint64_t> ids(x->B_max);
    std::vector<int> removed(1024);
    std::vector<slim_request> next_q;
    int finished = 0;
    while (finished < n) {
        if (slim_status sa = admit(now())) return sa;
        slim_sched_action act;
        // VRAM_used for CANLOAD (l.14): the caller's figure + the buffers of the live instances (slab,
        // out, workspace each), so M_max bounds the scale-up; buffers parked in the free list are reused
        // by the next instance without a new allocation and are not counted
        const size_t res_bytes = x->inst_res.size() * (2 * x->B_max * x->out_bytes + x->wsb);
        slim_status s = slim_sched_next(x->sched, now(), -1.f, vram_external + res_bytes, &act, slots.data(), ids.data());
        if (s) return s;
        st.loads += act.n_loaded;
        if (act.kind == SLIM_ACT_RUN) {
            Res *r;
            auto it = x->inst_res.find(act.inst);
            if (it != x->inst_res.end()) {
                r = it->second;
            } else {
                if (!x->free_res.empty()) {
                    r = x->free_res.back();
                    x->free_res.pop_back();
                } else if ((s = new_res(x, &r))) {
                    return s;
                }
                x->inst_res[act.inst] = r;
            }
            const int b = act.batch, seg = act.seg;
            std::memcpy(r->slots_h, slots.data(), b * sizeof(uint32_t));
            if (cudaMemcpyAsync(r->slots_d, r->slots_h, b * sizeof(uint32_t), cudaMemcpyHostToDevice, r->stream) !=
                cudaSuccess)
                return SLIM_ECUDA;
            slim_launch_desc d{seg, act.w_prev, act.w_req, b, 0};
            const void *pool = seg == 0 ? images : x->pools[seg];
            if ((s = slim_launch(x->ctx, &d, r->slots_d, pool, x->row_bytes[seg], r->slab, r->out, r->ws, x->wsb,
                                 r->stream)))
                return s;
            if (seg < 3) {
                const size_t h = static_cast<size_t>(c.image_hw >> seg);
                const size_t row = h * h * slim_act_channels(act.w_req, c.base_channels[seg]) * x->eb;
                s = slim_scatter(x->ctx, r->out, r->slots_d, b, row, x->pools[seg + 1], x->row_bytes[seg + 1], r->stream);
            } else {
                s = slim_scatter(x->ctx, r->out, r->slots_d, b, c.num_classes * 4, logits, c.num_classes * 4, r->stream);
            }
            if (s) return s;
            if (cudaEventRecord(r->event, r->stream) != cudaSuccess) return SLIM_ECUDA;
            pending.push_back(Pending{act.inst, seg, b, r, std::vector<uint64_t>(ids.begin(), ids.begin() + b)});
            st.batches += 1;
            continue;
        }
        if (act.kind == SLIM_ACT_REQUEUE) st.requeues += 1;
        if (pending.empty()) {   // nothing in flight: only the unloader can free capacity
            if (act.kind == SLIM_ACT_IDLE) {
                if (admitted >= n) return SLIM_EINVAL;   // queue empty with requests unfinished: cannot happen
                while (!arrival_due()) {
                }   // open loop: idle until the next arrival
                continue;
            }
            const int k = slim_sched_unload_idle(x->sched, now(), removed.data(), static_cast<int>(removed.size()));
            for (int i = 0; i < k && i < static_cast<int>(removed.size()); ++i) {
                auto it = x->inst_res.find(removed[i]);
                if (it != x->inst_res.end()) {
                    x->free_res.push_back(it->second);
                    x->inst_res.erase(it);
                }
            }
            st.unloaded += k;
            if (k == 0) {
                slim_instance inf[64];
                const int ni = slim_sched_instances(x->sched, inf, 64);
                if (ni == 0) return SLIM_ENOMEM;   // CANLOAD can never pass (M_max / U_blk): deadlock
            }
            continue;
        }
        // wait for whichever in-flight batch finishes first (or a new arrival), then release the finished
        for (bool any = false; !any;) {
            if (arrival_s && arrival_due()) break;
            for (const Pending &p : pending) {
                const cudaError_t e = cudaEventQuery(p.res->event);
                if (e == cudaSuccess) {
                    any = true;
                    break;
                }
                if (e != cudaErrorNotReady) return SLIM_ECUDA;
            }
        }
        const double t = now();
        for (size_t i = 0; i < pending.size();) {
            if (cudaEventQuery(pending[i].res->event) != cudaSuccess) {
                ++i;
                continue;
            }
            Pending p = std::move(pending[i]);
            pending.erase(pending.begin() + static_cast<long>(i));
            if ((s = slim_sched_complete(x->sched, p.inst, t))) return s;
            if (p.seg < 3) {
                next_q.clear();
                for (uint64_t id : p.ids)
                    next_q.push_back(slim_request{id, p.seg + 1, tuples[4 * id + p.seg + 1], tuples[4 * id + p.seg],
                                                  static_cast<uint32_t>(id)});
                if ((s = slim_sched_enqueue(x->sched, next_q.data(), static_cast<int>(next_q.size()), t))) return s;
            } else {
                finished += p.batch;
                if (done_s)
                    for (uint64_t id : p.ids) done_s[id] = t;
            }
        }
        const int k = slim_sched_unload_idle(x->sched, now(), removed.data(), static_cast<int>(removed.size()));
        for (int i = 0; i < k && i < static_cast<int>(removed.size()); ++i) {
            auto it = x->inst_res.find(removed[i]);
            if (it != x->inst_res.end()) {
                x->free_res.push_back(it->second);
                x->inst_res.erase(it);
            }
        }
        st.unloaded += k;
    }
    for (auto &kv : x->inst_res) cudaStreamSynchronize(kv.second->stream);
    st.seconds = now();
    if (stats) *stats = st;
    return slim_last_error(x->ctx);
}

}  // extern "C"
