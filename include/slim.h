/*
 * slim.h -- C-ABI of libslim.so: the batched forward pass of a segmented,
 * width-sliced SlimResNet on NVIDIA B200 (sm_100a).  This is the data-parallel
 * hot path of Slim Scheduler (arXiv 2510.09018); everything around it (PPO
 * router, greedy executor) is host-side control that calls these entry points.
 *
 * Citations: P:n = PAPER.md line n (the paper text); SURVEY §x = SURVEY.md.
 *   - segmented, universally slimmable backbone ............ P:31
 *   - request key k = (s, w_req, w_prev), batching by key ... P:49, Alg.1 l.4
 *   - RUNBATCH(inst, B) on a loaded (segment, width) ........ Alg.1 l.10
 *   - "Estimate bytes of (s, w)" (CANLOAD) .................. Alg.1 l.14
 *   - "offload to CPU, free VRAM" (UNLOADERLOOP) ............ Alg.1 l.25
 *   - widths W = {1.00, 0.75, 0.50, 0.25}, four segments .... P:148
 * The paper gives no depth, channel counts or normalisation details for its
 * kernels; DESIGN.md "Readings" lists how each silence is resolved (ResNet-18
 * CIFAR, switchable per-width BN selected by the segment's own width, eps, ...).
 *
 * Conventions (all entry points):
 *   - Return slim_status; nothing throws across the ABI.  Argument validation
 *     happens BEFORE anything is enqueued: on SLIM_EINVAL / SLIM_ENOTLOADED no
 *     work was launched.  Asynchronous device faults are sticky and surface as
 *     SLIM_ECUDA from the next call or from slim_last_error().
 *   - Device buffers (in, out, workspace, slab, pool, slots) are caller-owned
 *     device memory, 16-byte aligned.  The library never frees them and never
 *     allocates device memory inside forward / launch calls.
 *   - All device work is enqueued on the caller's `stream` (a cudaStream_t
 *     passed as void*; NULL = legacy default stream).  No implicit host sync.
 *   - Activations are dense NHWC.  In SLIM_BF16 mode activations are bf16
 *     (uint16 bit patterns) with fp32 accumulation and fp32 epilogue math and
 *     one bf16 rounding per stored tensor; in SLIM_FP32 mode they are fp32
 *     with fp32 FFMA (no TF32 anywhere).  Logits are always fp32.
 *   - Width semantics: a width r must be one of cfg.widths (|diff| < 1e-6);
 *     the active channel count of a C-channel layer is c(r, C) = ceil(r*C).
 *     The first ceil(r*C) output channels and the first c(r_prev) input
 *     channels of the FULL-width shared weights are used, selected by TMA
 *     tensor-map bounds (tile predication), never by copying weights.
 *   - Thread safety: after loading, forward calls on one context may run
 *     concurrently from several threads on different streams ONLY when each
 *     passes its own workspace (slim_forward_ws / slim_forward_chain);
 *     slim_forward uses the context's internal workspace and is not
 *     re-entrant.  Load/unload must not overlap forwards of the same segment.
 */
#ifndef SLIM_H_
#define SLIM_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SLIM_API __attribute__((visibility("default")))
#else
#define SLIM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SLIM_OK = 0,
    SLIM_EINVAL = -1,          /* bad argument (width not in set, seg out of range, B>B_max, misaligned ptr, ...) */
    SLIM_ENOTLOADED = -2,      /* segment not loaded (slim_load_segment) */
    SLIM_ENOMEM = -3,          /* device / host allocation failed at create or load */
    SLIM_ECUDA = -4,           /* CUDA runtime / driver error (sticky for async faults) */
    SLIM_EUNSUPPORTED = -5     /* configuration outside what the kernels implement */
} slim_status;

typedef enum { SLIM_BF16 = 0, SLIM_FP32 = 1 } slim_dtype;

/* Normalisation after every conv.  SLIM_NORM_BN: switchable inference BatchNorm per
 * width (north_star; folded into the conv epilogue).  SLIM_NORM_GN: GroupNorm, what the
 * paper's model uses ("Group Normalization instead of Batch Normalization to avoid
 * cross-width statistics drift"): statistics per
 * (image, group of gn_group_channels consecutive channels) over H*W*gn_group_channels
 * values, biased variance, bn_eps; affine gamma/beta per (layer, width) (slim_bn's
 * mean/var are not read and may be NULL).  DESIGN.md reading R16. */
typedef enum { SLIM_NORM_BN = 0, SLIM_NORM_GN = 1 } slim_norm;

/* Network configuration (reading D1 = CIFAR ResNet-18). */
typedef struct {
    int n_widths;              /* |W|, 1..8 */
    float widths[8];           /* sorted ascending, each in (0,1]; default {0.25,0.5,0.75,1.0};
                                  any values (universal widths, see slim_act_channels) */
    int blocks_per_seg[4];     /* BasicBlocks per segment, default {2,2,2,2} (1..4 each) */
    int base_channels[4];      /* full-width channels C_s, default {64,128,256,512} */
    int in_channels;           /* image channels, 3 (never sliced) */
    int num_classes;           /* classifier outputs, 100 for CIFAR-100; never sliced; <= 1024 */
    int image_hw;              /* input height = width, 32 */
    int max_batch;             /* B_max: bounds every batch; sizes the internal workspace */
    float bn_eps;              /* BatchNorm epsilon, 1e-5 */
    slim_dtype dtype;          /* SLIM_BF16 (default) or SLIM_FP32 */
    slim_norm norm;            /* SLIM_NORM_BN (default) or SLIM_NORM_GN */
    int gn_group_channels;     /* GN group size, default 16; a multiple of 8 dividing every c(r, C_s),
                                  else slim_create returns SLIM_EUNSUPPORTED */
} slim_config;

/* Host pointers to ONE segment's full-width weights, fp32 values (copied at load).
 * conv_w order (the manifest order):
 *   seg 0   : stem, then per block b: b.c1, b.c2
 *   seg s>0 : block 0: c1 (3x3 stride 2), c2, sc (1x1 stride 2 projection);
 *             blocks b>0: c1, c2
 * Each conv tensor is KRSC [C_out][k][k][C_in] at full width.  fc_w [classes][C_3]
 * and fc_b [classes] are read for seg 3 only (may be NULL otherwise). */
typedef struct {
    const float *conv_w[16];
    int n_conv;
    const float *fc_w;
    const float *fc_b;
} slim_seg_weights;

/* Inference BatchNorm statistics of one layer at one width; each array has
 * c(width, C_out) entries.  z = (y - mean)/sqrt(var + eps)*gamma + beta. */
typedef struct { const float *gamma, *beta, *mean, *var; } slim_bn;

/* The BN statistics of every conv layer of one segment (manifest order) at one width. */
typedef struct { const slim_bn *per_layer; int n_layers; } slim_bn_set;

typedef struct slim_ctx slim_ctx;

/* ---- lifetime ---------------------------------------------------------- */

/* Create a context on CUDA device `device`; validates cfg and allocates the
 * internal workspace for cfg->max_batch.  *out = NULL on failure. */
SLIM_API slim_status slim_create(int device, const slim_config *cfg, slim_ctx **out);
SLIM_API void slim_destroy(slim_ctx *ctx);
/* Fill *cfg with the defaults above (B_max = 4096, SLIM_BF16). */
SLIM_API void slim_default_config(slim_config *cfg);

/* Load segment `seg` (0..3): copies the full-width weights to the device
 * (bf16 RNE in BF16 mode), folds every width's BN into fp32 (scale, shift) in
 * fp64 on the host, and encodes the weight tensor maps for every (r_prev, r).
 * bn_per_width points to cfg.n_widths sets (one per width, same order as
 * cfg.widths).  Replaces a previously loaded copy.  Synchronous. */
SLIM_API slim_status slim_load_segment(slim_ctx *ctx, int seg, const slim_seg_weights *w,
                              const slim_bn_set *bn_per_width);
/* Alg.1 UNLOADERLOOP: free the segment's device memory. */
SLIM_API slim_status slim_unload_segment(slim_ctx *ctx, int seg);
SLIM_API int slim_segment_loaded(const slim_ctx *ctx, int seg);

/* CANLOAD's "Estimate bytes of (s, w)": device bytes of the ACTIVE
 * weights and folded BN of segment seg at (r_prev, r) in cfg->dtype (the
 * resident copy is full-width; this is the slice a width-r instance reads). */
SLIM_API size_t slim_segment_bytes(const slim_config *cfg, int seg, float r_prev, float r);

/* ---- forward ----------------------------------------------------------- */

/* RUNBATCH (Alg.1 l.10) for one segment at key (seg, r, r_prev):
 *   in : seg 0: [B, H, H, in_channels]; seg s>0: [B, H_{s-1}, H_{s-1}, c_{s-1}(r_prev)]
 *   out: seg < 3: [B, H_s, H_s, c_s(r)]; seg 3: fp32 logits [B, num_classes]
 * H_s = image_hw / 2^s.  r_prev is ignored for seg 0.  1 <= B <= max_batch.
 * Uses the context's internal workspace (not re-entrant; see slim_forward_ws). */
SLIM_API slim_status slim_forward(slim_ctx *ctx, int seg, float r_prev, float r, int batch,
                         const void *in, void *out, void *stream);
SLIM_API size_t slim_forward_workspace_bytes(const slim_ctx *ctx, int seg, float r_prev, float r, int batch);
SLIM_API slim_status slim_forward_ws(slim_ctx *ctx, int seg, float r_prev, float r, int batch,
                            const void *in, void *out, void *ws, size_t ws_bytes, void *stream);

/* The whole chain seg0(r0) -> seg1(r0->r1) -> seg2(r1->r2) -> seg3(r2->r3) -> head,
 * i.e. the composition of slim_forward calls (P:49 re-entry with w_prev).
 * in: [B, H, H, in_channels]; logits: fp32 [B, num_classes]; ws: device workspace
 * of at least slim_chain_workspace_bytes(). */
SLIM_API size_t slim_chain_workspace_bytes(const slim_ctx *ctx, const float r_per_seg[4], int batch);
SLIM_API slim_status slim_forward_chain(slim_ctx *ctx, const float r_per_seg[4], int batch, const void *in,
                               float *logits, void *ws, size_t ws_bytes, void *stream);

/* ---- batch packer (Alg.1 l.3-4) --------------------------------- */

/* One queued request: key (seg, w_req, w_prev).  `slot` is the row
 * of this request's input activation in the caller's activation pool. */
typedef struct {
    uint64_t id;
    int seg;
    float w_req;
    float w_prev;              /* ignored when seg == 0 */
    uint32_t slot;
} slim_request;

/* One batch of key-equal requests: order[first .. first+batch) (written by
 * slim_pack) are the request indices, FIFO order preserved. */
typedef struct {
    int seg;
    float r_prev;
    float r;
    int batch;
    int first;
} slim_launch_desc;

/* Greedy key batching over the FIFO q[0..n): repeatedly peek the head key,
 * take up to B_max requests with an equal key scanning the whole queue
 * (non-matching requests keep their relative order, SPEC form_batch), and emit
 * one descriptor.  Host only.  order: n entries; descs: capacity max_descs
 * (n suffices).  Keys are validated against cfg's widths (SLIM_EINVAL).  Needs no GPU. */
SLIM_API slim_status slim_pack(const slim_config *cfg, const slim_request *q, int n, int B_max,
                      slim_launch_desc *descs, int max_descs, int *n_descs, uint32_t *order);

/* Run one packed batch: gather rows pool[slots[i]] (each pool_row_bytes, device)
 * into the contiguous slab (device, >= batch rows) with the vectorised gather
 * kernel, then slim_forward_ws on the slab into out.  slots is a DEVICE array of
 * desc->batch uint32 row indices; if slots == NULL the pool is already the
 * contiguous batch and no gather runs. */
SLIM_API slim_status slim_launch(slim_ctx *ctx, const slim_launch_desc *desc, const uint32_t *slots,
                        const void *pool, size_t pool_row_bytes, void *slab, void *out,
                        void *ws, size_t ws_bytes, void *stream);

/* Device gather alone (K8): dst[i] = src[idx[i]] for i < n rows of row_bytes
 * (multiple of 16).  idx is a device array. */
SLIM_API slim_status slim_gather(slim_ctx *ctx, const void *src, const uint32_t *idx, int n, size_t row_bytes,
                        void *dst, void *stream);

/* Device scatter (inverse of slim_gather): row i of src (row_bytes, multiple of 16)
 * goes to dst + idx[i]*dst_stride; used to return a packed batch's outputs to the
 * per-request activation pool of the next segment (P:49 re-entry with w_prev). */
SLIM_API slim_status slim_scatter(slim_ctx *ctx, const void *src, const uint32_t *idx, int n, size_t row_bytes,
                                  void *dst, size_t dst_stride, void *stream);

/* ---- Algorithm 1: greedy segment-slim scheduler (host) ----
 * A per-server decision engine: FIFO queue of requests keyed (s, w_req, w_prev), batch
 * formation from the head key (l.3-4), FINDFREEBESTFIT (l.5, l.11-12: free instance of
 * segment s with the smallest width >= w_req), CANLOAD (l.7, l.13-20: VRAM cap M_max and
 * utilisation gate U_blk), the opportunistic scale-up of P:49 (up to N_new instances of
 * key k when its queue holds >= Q_th requests, else one; each guarded by CANLOAD),
 * requeue-to-front on failure (l.9) and UNLOADERLOOP (l.21-25: non-busy instances idle
 * >= t_idle are removed).  Host only, no CUDA calls, thread-safe (one mutex).  An
 * "instance" is an execution slot (the caller gives each one a CUDA stream); its
 * bytes are slim_segment_bytes(cfg, s, w, w), and VRAM_used = vram_external (passed by
 * the caller) + the bytes of the live instances (reading R17). */
typedef struct {
    int B_max;                 /* batch limit */
    double M_max_bytes;        /* VRAM cap M_max (bytes) */
    float U_blk;               /* utilisation block threshold, fraction in [0, 1] */
    double t_idle_s;           /* idle-unload time t_idle (s) */
    int Q_th;                  /* scale trigger: key-k queue length that scales up by N_new */
    int N_new;                 /* scale cap: instances added per scale-up */
} slim_sched_knobs;
typedef struct slim_sched slim_sched;
typedef enum { SLIM_ACT_IDLE = 0, SLIM_ACT_RUN = 1, SLIM_ACT_REQUEUE = 2 } slim_sched_act_kind;
typedef struct {
    int kind;                  /* slim_sched_act_kind: IDLE = queue empty; REQUEUE = no instance (l.9) */
    int inst;                  /* RUN: instance id (busy until slim_sched_complete) */
    int seg;                   /* the batch key (s, w_req, w_prev) (w_prev = 0 for seg 0) */
    float w_req, w_prev;
    float inst_w;              /* RUN: the instance's width (>= w_req; compute follows w_req, R9) */
    int batch;                 /* RUN: requests taken; their slots/ids are written in FIFO order */
    int n_loaded;              /* instances created by this call (CANLOAD passed) */
} slim_sched_action;
typedef struct {
    int id, seg;
    float w;
    int busy;
    double t_last;
    size_t bytes;
} slim_instance;
/* Defaults: B_max 256, M_max 64e9 B (the paper's 64 GB devices), U_blk 0.95,
 * t_idle 1 s, Q_th 512, N_new 2 (the paper gives no values; all knobs). */
SLIM_API void slim_sched_default_knobs(slim_sched_knobs *k);
SLIM_API slim_status slim_sched_create(const slim_config *cfg, const slim_sched_knobs *knobs, slim_sched **out);
SLIM_API void slim_sched_destroy(slim_sched *s);
/* Append n requests (key validated against cfg's widths; SLIM_EINVAL leaves Q unchanged). */
SLIM_API slim_status slim_sched_enqueue(slim_sched *s, const slim_request *reqs, int n, double t_enq);
/* One LOOP iteration at time `now` (s).  util: latest utilisation sample in [0,1], or < 0
 * for none (l.18 "u != empty").  slots (and ids if non-NULL) must hold B_max entries. */
SLIM_API slim_status slim_sched_next(slim_sched *s, double now, float util, size_t vram_external,
                                     slim_sched_action *act, uint32_t *slots, uint64_t *ids);
/* RUNBATCH finished on instance inst: busy = false, t_last = now. */
SLIM_API slim_status slim_sched_complete(slim_sched *s, int inst, double now);
/* UNLOADERLOOP pass: removes idle instances, writes up to max_removed ids, returns the count. */
SLIM_API int slim_sched_unload_idle(slim_sched *s, double now, int *removed, int max_removed);
SLIM_API int slim_sched_queue_len(const slim_sched *s);
/* The scheduler's batch cap (knobs.B_max): the most slots/ids one slim_sched_next writes. */
SLIM_API int slim_sched_b_max(const slim_sched *s);
/* Copies up to max_out instance records; returns the number of live instances. */
SLIM_API int slim_sched_instances(const slim_sched *s, slim_instance *out, int max_out);

/* ---- native Alg. 1 executor (one GPU) ------------------------------------------------
 * Drives the scheduler's LOOP in C++: each RUN decision copies the batch's slots to the
 * device and runs slim_launch (gather + segment) and slim_scatter (outputs -> the next
 * segment's request pool, or the logits) on the instance's own CUDA stream; finished
 * batches (event polling) release their instance and re-enqueue their requests with key
 * (s+1, w_{s+1}, w_s); idle instances are unloaded (their buffers are recycled).
 * create: allocates the per-segment request pools for n_max requests; the scheduler
 * stays owned by the caller; SLIM_EINVAL unless slim_sched_b_max(sched) <= B_max <= cfg.max_batch
 * (every buffer is sized for B_max requests per batch).  run: images = device
 * [n][H][W][in_channels]; tuples = HOST float [n][4] (the width of each segment, each in
 * cfg.widths); logits = device fp32 [n][num_classes]; vram_external as in slim_sched_next, to which
 * the executor adds the buffers of its live instances (slab, out, workspace: M_max bounds scale-up);
 * the call returns when every request is done (stream: ordered before the first read).
 * arrival_s (host, n, ascending, may be NULL): open loop -- request i enters the queue once the
 * loop's clock (s since the call began) reaches arrival_s[i]; NULL = all at t = 0 (closed loop).
 * done_s (host, n, may be NULL): the clock when request i's segment-3 batch was seen complete. */
typedef struct slim_exec slim_exec;
typedef struct {
    int batches, loads, requeues, unloaded;
    double seconds;            /* host wall time of the loop */
} slim_exec_stats;
SLIM_API slim_status slim_exec_create(slim_ctx *ctx, slim_sched *sched, int n_max, int B_max, slim_exec **out);
SLIM_API void slim_exec_destroy(slim_exec *x);
SLIM_API slim_status slim_exec_run(slim_exec *x, const void *images, const float *tuples, int n, float *logits,
                                   size_t vram_external, slim_exec_stats *stats, void *stream,
                                   const double *arrival_s, double *done_s);

/* ---- native request-stream executor (CFG4; Alg. 1 l.3-4 + l.10) ----------------
 * One call runs a whole request stream through the four segments with the key batching of
 * slim_pack (FIFO head key, up to B_max equal keys, per segment with key (s, w_s, w_{s-1}))
 * and, per batch, slim_launch (gather + segment kernels) and slim_scatter (outputs -> the
 * next segment's request pool, or the logits).  All four packings are done on the host
 * first (they depend only on the tuples); the four request orders go to the device in ONE
 * H2D copy from a double-buffered pinned staging area.  lanes > 1: the batches of one
 * segment run on `lanes` streams (lane = width index, plus a rotation over a width's batches
 * when lanes > widths), forked from and joined back to the caller's stream around each
 * segment; the per-width SM shares of slim_set_sm_share keep them side by side.
 * create: allocates the pools for n_max requests and per-lane slab/out/workspace buffers for
 * B_max rows (SLIM_EINVAL unless 1 <= B_max <= cfg.max_batch, 1 <= lanes <= 16).
 * run: images = device [n][H][W][in_channels] (activation dtype); tuples = HOST float [n][4]
 * (each in cfg.widths, else SLIM_EINVAL before any launch); logits = device fp32
 * [n][num_classes].  Asynchronous: everything is ordered on `stream` (and after what was
 * enqueued on it before the call); the call returns after enqueueing.  The host blocks only
 * when a staging buffer is still being read by the copy of the call before the previous one.
 * stats (may be NULL): batches, kernels launched, host seconds spent packing and in the whole call
 * (incl. any wait for the staging buffer). */
typedef struct slim_stream slim_stream;
typedef struct {
    int batches;               /* packed batches over the four segments */
    int launches;              /* kernels this call launched (gather, segment kernels, scatter) */
    double pack_seconds;       /* host: the four slim_pack calls */
    double host_seconds;       /* host: the whole call (pack + staging + enqueueing) */
} slim_stream_stats;
SLIM_API slim_status slim_stream_create(slim_ctx *ctx, int n_max, int B_max, int lanes, slim_stream **out);
SLIM_API void slim_stream_destroy(slim_stream *x);
SLIM_API slim_status slim_stream_run(slim_stream *x, const void *images, const float *tuples, int n, float *logits,
                                     void *stream, slim_stream_stats *stats);

/* ---- execution modes and profiling ------------------------------------- */

/* Graph mode (default off): slim_forward_ws / slim_forward_chain capture their
 * launch sequence into a CUDA graph the first time a given argument list
 * (key, batch, buffer pointers) is seen and replay it afterwards -- one
 * cudaGraphLaunch per call instead of ~18 kernel launches.  Captured graphs
 * bake in the buffer addresses; loading/unloading a segment drops them. */
SLIM_API slim_status slim_set_graph_mode(slim_ctx *ctx, int enable);

/* SM partitioning for concurrent width instances: every persistent kernel this context launches
 * for width r uses at most round(share * num_SMs) CTAs (share in (0,1]; default 1 = all SMs).
 * At small batches the kernels are latency chains that each occupy every SM with one CTA, so
 * instances of different widths on different streams serialise kernel by kernel; disjoint SM
 * shares let them run side by side.  Synchronises the device and drops the
 * captured graphs.  SLIM_EINVAL if r is not a configured width or share is outside (0,1]. */
SLIM_API slim_status slim_set_sm_share(slim_ctx *ctx, float r, float share);

/* Per-launch profiling: while on, every kernel launch is bracketed by CUDA
 * events on its stream and described by its algorithmic work (SURVEY §8(d):
 * sliced FLOPs = 2*MACs; bytes = layer-materialised traffic: input, weights,
 * residual / projection input read once, output written once).  Graph replay
 * is bypassed while profiling.  begin() allocates the events (at most
 * max_launches records); end() synchronises and returns the records. */
typedef enum { SLIM_K_STEM = 0, SLIM_K_CONV_UMMA = 1, SLIM_K_HEAD = 2, SLIM_K_GATHER = 3, SLIM_K_CONV_F32 = 4,
               SLIM_K_GN = 5 /* GroupNorm apply (SLIM_NORM_GN) */,
               SLIM_K_SEG_FUSED = 6 /* a whole segment in one kernel (narrow widths) */ } slim_kernel_kind;
typedef struct {
    int kind;                  /* slim_kernel_kind */
    int seg, layer;            /* segment, manifest index of the conv (stem = 0 in seg 0; head/gather: -1) */
    int batch;
    float r_prev, r;
    double flops, bytes;       /* algorithmic work of this launch */
    float ms;                  /* event-measured duration */
} slim_profile_record;
SLIM_API slim_status slim_profile_begin(slim_ctx *ctx, int max_launches);
SLIM_API slim_status slim_profile_end(slim_ctx *ctx, slim_profile_record *out, int max_out, int *n_out);

/* ---- errors, introspection ------------------------------------------------ */
SLIM_API slim_status slim_last_error(slim_ctx *ctx);        /* sticky async error (SLIM_OK if none) */
SLIM_API const char *slim_last_error_msg(const slim_ctx *ctx);
SLIM_API const char *slim_status_str(slim_status s);
SLIM_API int slim_version(void);
/* Number of kernels this context has launched (the bench's gpu_launches). */
SLIM_API uint64_t slim_launch_count(const slim_ctx *ctx);
/* Number of SMs of the context's device and the active-channel rule c(r, C). */
SLIM_API int slim_num_sms(const slim_ctx *ctx);
SLIM_API int slim_channels(float r, int C);
/* Universal widths ("universally slimmable"): any width in (0, 1]
 * may be configured.  Activations of width r carry c_act(r, C) = slim_act_channels(r, C)
 * channels per pixel: c(r, C) rounded up to a multiple of 16, and above 128 to a multiple of
 * 64 (the kernels' tile granules).  Channels c .. c_act-1 are exact zeros on output and are
 * ignored (multiply zero) on input.  For the paper's width set c_act == c. */
SLIM_API int slim_act_channels(float r, int C);

#ifdef __cplusplus
}
#endif
#endif /* SLIM_H_ */
