// slim_sched.cpp -- Algorithm 1 of the paper, the greedy segment-slim scheduler of one
// server, as a host-side decision engine.
//
// Host C++ only: no CUDA call is made here, so the scheduler is exercised on CPU by the
// tests; the caller (paper_2510_09018_b200/executor.py) executes each RUN decision on
// the GPU through slim_launch on the instance's stream and reports completion.
//
//   LOOP (l.1-10):  peek the FIFO head key (s, w_req, w_prev); form a batch of up to
//                   B_max requests of that key; inst = FINDFREEBESTFIT (free instance of
//                   segment s with minimal width >= w_req); if none, CANLOAD / scale up;
//                   if still none, requeue the batch to the FRONT of Q; else RUN.
//   CANLOAD (l.13-20): bytes of (s, w) = slim_segment_bytes(cfg, s, w, w);
//                   VRAM_used + bytes > M_max -> no; latest util >= U_blk -> no.
//   scale-up: "instantiating up to N_new additional instances for key k" when no
//                   instance fits -- reading R17: N_new instances when the queued count of
//                   key k is >= Q_th (the scale trigger), else one; each guarded by CANLOAD.
//   UNLOADERLOOP (l.21-25): non-busy instances idle for >= t_idle are removed.
//
// VRAM_used (reading R17) = the caller's external usage + the bytes of this scheduler's
// live instances, so decisions are a deterministic function of the call sequence.
#include <cstdint>
#include <cstring>
#include <deque>
#include <mutex>
#include <vector>

#include "../../include/slim.h"

namespace {

struct QEntry {
    slim_request r;
    double t_enq;
    int64_t seq;   // global FIFO position (requeued batches get positions before every other entry)
};

// The FIFO queue Q, held as one FIFO per key (there are at most 4 + 16*3 keys): the head key is
// the key whose oldest entry has the smallest sequence number, so a LOOP step costs O(keys + B)
// instead of a pass over the whole queue; global FIFO order is the sequence order.
struct KeyQ {
    slim_request key;
    std::deque<QEntry> q;
};

struct Inst {
    int id, seg;
    float w;
    bool busy;
    double t_last;
    size_t bytes;
};

bool same_w(float a, float b) { return a - b < 1e-6f && b - a < 1e-6f; }

int width_idx(const slim_config &c, float r) {
    for (int i = 0; i < c.n_widths; ++i)
        if (same_w(c.widths[i], r)) return i;
    return -1;
}

bool key_eq(const slim_request &a, const slim_request &b) {
    return a.seg == b.seg && same_w(a.w_req, b.w_req) && (a.seg == 0 || same_w(a.w_prev, b.w_prev));
}

}  // namespace

struct slim_sched {
    slim_config cfg{};
    slim_sched_knobs k{};
    std::mutex mu;
    std::vector<KeyQ> keys;
    int64_t next_seq = 0, front_seq = -1;
    size_t total = 0;
    KeyQ &key_queue(const slim_request &r) {
        for (KeyQ &k : keys)
            if (key_eq(k.key, r)) return k;
        keys.push_back(KeyQ{r, {}});
        return keys.back();
    }
    std::vector<Inst> inst;
    int next_id = 0;
    size_t live_bytes() const {
        size_t b = 0;
        for (const Inst &i : inst) b += i.bytes;
        return b;
    }
    // CANLOAD(s, w) (l.13-20): the VRAM cap and the utilisation gate
    bool can_load(int seg, float w, size_t vram_external, float util, size_t *bytes) const {
        *bytes = slim_segment_bytes(&cfg, seg, w, w);
        if (static_cast<double>(vram_external + live_bytes() + *bytes) > k.M_max_bytes) return false;
        if (util >= 0.f && util >= k.U_blk) return false;
        return true;
    }
    // FINDFREEBESTFIT (l.11-12): free instance of segment s with minimal width >= w_req
    int best_fit(int seg, float w_req) const {
        int best = -1;
        for (size_t i = 0; i < inst.size(); ++i) {
            const Inst &x = inst[i];
            if (x.busy || x.seg != seg || x.w < w_req - 1e-6f) continue;
            if (best < 0 || x.w < inst[best].w) best = static_cast<int>(i);
        }
        return best;
    }
};

extern "C" {

void slim_sched_default_knobs(slim_sched_knobs *k) {
    std::memset(k, 0, sizeof *k);
    k->B_max = 256;
    k->M_max_bytes = 64e9;   // the paper's devices report 64 GB; a knob
    k->U_blk = 0.95f;        // utilisation fraction (R13: SI units)
    k->t_idle_s = 1.0;
    k->Q_th = 512;
    k->N_new = 2;
}

slim_status slim_sched_create(const slim_config *cfg, const slim_sched_knobs *knobs, slim_sched **out) {
    if (!out) return SLIM_EINVAL;
    *out = nullptr;
    if (!cfg || !knobs || knobs->B_max < 1 || knobs->N_new < 1 || knobs->Q_th < 1 || !(knobs->M_max_bytes > 0) ||
        knobs->t_idle_s < 0 || cfg->n_widths < 1 || cfg->n_widths > 8)
        return SLIM_EINVAL;
    slim_sched *s = new slim_sched();
    s->cfg = *cfg;
    s->k = *knobs;
    *out = s;
    return SLIM_OK;
}

void slim_sched_destroy(slim_sched *s) { delete s; }

slim_status slim_sched_enqueue(slim_sched *s, const slim_request *reqs, int n, double t_enq) {
    if (!s || n < 0 || (n > 0 && !reqs)) return SLIM_EINVAL;
    for (int i = 0; i < n; ++i) {   // validate everything before changing the queue
        const slim_request &r = reqs[i];
        if (r.seg < 0 || r.seg > 3 || width_idx(s->cfg, r.w_req) < 0 ||
            (r.seg > 0 && width_idx(s->cfg, r.w_prev) < 0))
            return SLIM_EINVAL;
    }
    std::lock_guard<std::mutex> g(s->mu);
    for (int i = 0; i < n; ++i) {
        s->key_queue(reqs[i]).q.push_back(QEntry{reqs[i], t_enq, s->next_seq++});
        ++s->total;
    }
    return SLIM_OK;
}

slim_status slim_sched_next(slim_sched *s, double now, float util, size_t vram_external, slim_sched_action *act,
                            uint32_t *slots, uint64_t *ids) {
    if (!s || !act || !slots) return SLIM_EINVAL;
    std::lock_guard<std::mutex> g(s->mu);
    std::memset(act, 0, sizeof *act);
    act->inst = -1;
    if (s->total == 0) {   // l.3 "wait until Q non-empty": the caller waits
        act->kind = SLIM_ACT_IDLE;
        return SLIM_OK;
    }
    // l.3-4: head key = the key of the oldest request; batch = its first B_max requests (FIFO order)
    KeyQ *hq = nullptr;
    for (KeyQ &k : s->keys)
        if (!k.q.empty() && (!hq || k.q.front().seq < hq->q.front().seq)) hq = &k;
    const slim_request head = hq->q.front().r;
    const int key_count = static_cast<int>(hq->q.size());
    const int nb = key_count < s->k.B_max ? key_count : s->k.B_max;
    act->seg = head.seg;
    act->w_req = head.w_req;
    act->w_prev = head.seg ? head.w_prev : 0.f;
    // l.5: best fit among free instances
    int bi = s->best_fit(head.seg, head.w_req);
    if (bi < 0) {
        // l.6-7 CANLOAD, with the opportunistic scale-up: up to N_new instances of key k when
        // the key's queue is at least the scale trigger Q_th, else one
        const int want = key_count >= s->k.Q_th ? s->k.N_new : 1;
        for (int j = 0; j < want; ++j) {
            size_t bytes = 0;
            if (!s->can_load(head.seg, head.w_req, vram_external, util, &bytes)) break;
            s->inst.push_back(Inst{s->next_id++, head.seg, head.w_req, false, now, bytes});
            ++act->n_loaded;
        }
        if (act->n_loaded) bi = static_cast<int>(s->inst.size()) - act->n_loaded;   // first new instance
    }
    if (bi < 0) {   // l.8-9: requeue B to the front of Q (batch order, then the rest)
        const int64_t base = s->front_seq - nb + 1;
        for (int i = 0; i < nb; ++i) hq->q[i].seq = base + i;
        s->front_seq = base - 1;
        act->kind = SLIM_ACT_REQUEUE;
        act->batch = nb;
        return SLIM_OK;
    }
    // l.10: mark busy, hand the batch to the caller (RUNBATCH)
    Inst &I = s->inst[bi];
    I.busy = true;
    I.t_last = now;
    act->kind = SLIM_ACT_RUN;
    act->inst = I.id;
    act->inst_w = I.w;
    act->batch = nb;
    for (int i = 0; i < nb; ++i) {
        const QEntry &e = hq->q.front();
        slots[i] = e.r.slot;
        if (ids) ids[i] = e.r.id;
        hq->q.pop_front();
    }
    s->total -= nb;
    return SLIM_OK;
}

slim_status slim_sched_complete(slim_sched *s, int inst_id, double now) {
    if (!s) return SLIM_EINVAL;
    std::lock_guard<std::mutex> g(s->mu);
    for (Inst &I : s->inst)
        if (I.id == inst_id) {
            if (!I.busy) return SLIM_EINVAL;
            I.busy = false;
            I.t_last = now;   // l.10 "update inst.t_last"
            return SLIM_OK;
        }
    return SLIM_EINVAL;
}

int slim_sched_unload_idle(slim_sched *s, double now, int *removed, int max_removed) {
    if (!s) return -1;
    std::lock_guard<std::mutex> g(s->mu);
    int n = 0;
    std::vector<Inst> keep;
    for (const Inst &I : s->inst) {
        if (!I.busy && now - I.t_last >= s->k.t_idle_s) {   // l.23-25
            if (removed && n < max_removed) removed[n] = I.id;
            ++n;
        } else {
            keep.push_back(I);
        }
    }
    s->inst.swap(keep);
    return n;
}

int slim_sched_b_max(const slim_sched *s) { return s ? s->k.B_max : 0; }

int slim_sched_queue_len(const slim_sched *s) {
    if (!s) return -1;
    std::lock_guard<std::mutex> g(const_cast<slim_sched *>(s)->mu);
    return static_cast<int>(s->total);
}

int slim_sched_instances(const slim_sched *s, slim_instance *out, int max_out) {
    if (!s) return -1;
    std::lock_guard<std::mutex> g(const_cast<slim_sched *>(s)->mu);
    const int n = static_cast<int>(s->inst.size());
    for (int i = 0; i < n && i < max_out && out; ++i) {
        const Inst &I = s->inst[i];
        out[i] = slim_instance{I.id, I.seg, I.w, I.busy ? 1 : 0, I.t_last, I.bytes};
    }
    return n;
}

}  // extern "C"
