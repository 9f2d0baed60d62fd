// slim_api.cu -- the C-ABI (include/slim.h): context, weight store, BN fold,
// tensor-map cache, segment/chain sequencing, batch packer and launcher.
//
// Host-side only; every arithmetic step of the forward pass runs in the kernels
// of kernels_umma.cu / kernels_simt.cu.  Citations: P:n = PAPER.md line n.
#include "slim_internal.h"

#include "../../include/slim.h"

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

using namespace slim;

namespace {

constexpr int kMaxLayers = 16;
constexpr int kMaxW = 8;

typedef CUresult (*PFN_encodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                    const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

struct LayerShape {
    int cout, cin, k, stride;
    bool is_stem, reads_prev;   // reads_prev: input width is the previous segment's (block 0 c1 / sc of seg>0)
};

struct DevLayer {
    LayerShape sh{};
    void *w = nullptr;                       // full-width KRSC, bf16 (BF16 mode) or fp32; stem: fp32
    float *scale[kMaxW] = {};                // folded BN per width, length c(width, cout)
    float *shift[kMaxW] = {};
    float *gn_gamma[kMaxW] = {};             // GroupNorm mode: affine per width (scale/shift are then the identity)
    float *gn_beta[kMaxW] = {};
    CUtensorMap tm[kMaxW][kMaxW][17];        // weight tensor map per (r_prev idx, r idx, n_tile/16)
    bool tm_ok[kMaxW][kMaxW][17] = {};
    CUtensorMap tmh[kMaxW][9][2];            // halo-kernel weight maps per (r idx, n_tile/16 - 1 (<=128), taps 3|9)
    bool tmh_ok[kMaxW][9][2] = {};
    void *stem_b = nullptr;                  // stem: the UMMA B operand image (64 rows x 128 B, SW128, bf16, K zero-padded)
    CUtensorMap tms[kMaxW][kMaxW];           // split-K kernel weight maps (64-channel boxes) per (r_prev idx, r idx)
    bool tms_ok[kMaxW][kMaxW] = {};
};

struct DevSegment {
    bool loaded = false;
    int n_conv = 0;
    DevLayer L[kMaxLayers];
    void *fimg[kMaxW][kMaxW] = {};           // fused-segment weight image per (r_prev idx, r idx) (seg >= 1)
    float *fc_w = nullptr, *fc_b = nullptr;
};

}  // namespace

struct slim_ctx {
    int device = 0;
    slim_config cfg{};
    int num_sms = 148;
    DevSegment seg[4];
    void *ws = nullptr;
    size_t ws_bytes = 0;
    std::atomic<uint64_t> launches{0};
    slim_status sticky = SLIM_OK;
    std::string msg;
    PFN_encodeTiled encode = nullptr;
    std::mutex mu;   // guards the lazily filled tensor-map cache
    // profiling: an event pair around every launch while prof_on
    bool prof_on = false;
    std::vector<cudaEvent_t> prof_ev;
    std::vector<slim_profile_record> prof_rec;
    // graph mode: captured launch sequences keyed by the full argument list
    struct GraphEntry {
        cudaGraphExec_t exec;
        uint64_t n_kernels;
    };
    bool graph_mode = false;
    // programmatic dependent launch between consecutive kernels (off while profiling); SLIM_PDL=0 (A/B)
    bool pdl = !getenv("SLIM_PDL") || atoi(getenv("SLIM_PDL")) != 0;
    cudaStream_t cap_stream = nullptr;
    std::mutex graph_mu;
    std::unordered_map<std::string, GraphEntry> graphs;
    unsigned long long *trace = nullptr;   // diagnostics: SLIM_CONV_TRACE -> per-CTA timestamps of the last conv
    float sm_share[8] = {1.f, 1.f, 1.f, 1.f, 1.f, 1.f, 1.f, 1.f};   // per width: persistent-grid cap / num_SMs
    std::mutex tm_mu;                                        // encoded tensor-map cache (encode_map)
    std::unordered_map<std::string, CUtensorMap> tm_cache;
};

namespace slim {
const slim_config *ctx_config(const slim_ctx *ctx) { return &ctx->cfg; }
}  // namespace slim

extern "C" int slim_channels(float r, int C) {
    // c(r, C) = ceil(r*C) (north_star); integer form for r = k/4 (exact for the width set of P:148)
    const double q = static_cast<double>(r) * 4.0;
    if (std::fabs(q - std::round(q)) < 1e-6) return (static_cast<int>(std::lround(q)) * C + 3) / 4;
    return static_cast<int>(std::ceil(static_cast<double>(r) * C - 1e-9));
}

// Universal widths ("universally slimmable"): activations and kernels
// use c_act(r, C) >= c(r, C) channels -- c rounded up to a multiple of 16 (the UMMA N / K-block
// granule) and, above 128, to a multiple of 64 (the N tiles of the conv kernels) -- and channels
// c .. c_act-1 are EXACT zeros: their folded BN scale/shift (GN: identity scale, gamma, beta) are
// zero, so conv outputs there are 0*acc + 0, and as inputs they multiply weights by zero.  For the
// paper's width set every c is already such a value (c_act == c).
extern "C" int slim_act_channels(float r, int C) {
    const int c = slim_channels(r, C);
    const int p16 = (c + 15) / 16 * 16;
    return p16 <= 128 ? p16 : (c + 63) / 64 * 64;
}

namespace {

slim_status fail(slim_ctx *ctx, slim_status s, const char *fmt, ...) __attribute__((format(printf, 3, 4)));
slim_status fail(slim_ctx *ctx, slim_status s, const char *fmt, ...) {
    if (ctx) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        ctx->msg = buf;
        if (s == SLIM_ECUDA) ctx->sticky = SLIM_ECUDA;
    }
    return s;
}

int width_index(const slim_config &c, float r) {
    for (int i = 0; i < c.n_widths; ++i)
        if (std::fabs(c.widths[i] - r) < 1e-6f) return i;
    return -1;
}

int seg_hw(const slim_config &c, int s) { return c.image_hw >> s; }
size_t elem_bytes(const slim_config &c) { return c.dtype == SLIM_BF16 ? 2 : 4; }
size_t round256(size_t x) { return (x + 255) & ~size_t(255); }
bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Manifest of one segment's conv layers (include/slim.h, slim_seg_weights).
int segment_layers(const slim_config &c, int s, LayerShape *out) {
    int n = 0;
    const int C = c.base_channels[s];
    if (s == 0) out[n++] = LayerShape{C, c.in_channels, 3, 1, true, false};
    for (int b = 0; b < c.blocks_per_seg[s]; ++b) {
        const bool down = (s > 0 && b == 0);
        const int cin = down ? c.base_channels[s - 1] : C;
        out[n++] = LayerShape{C, cin, 3, down ? 2 : 1, false, down};
        out[n++] = LayerShape{C, C, 3, 1, false, false};
        if (down) out[n++] = LayerShape{C, cin, 1, 2, false, true};
    }
    return n;
}

// index of block b's (c1, c2, sc) in the manifest
struct BlockIdx {
    int c1, c2, sc;
};
BlockIdx block_layers(const slim_config &c, int s, int b) {
    int i = (s == 0) ? 1 : 0;
    for (int bb = 0; bb < b; ++bb) i += (s > 0 && bb == 0) ? 3 : 2;
    BlockIdx r{i, i + 1, (s > 0 && b == 0) ? i + 2 : -1};
    return r;
}

size_t act_bytes(const slim_config &c, int s, float r, int B) {
    const int H = seg_hw(c, s);
    return static_cast<size_t>(B) * H * H * slim_act_channels(r, c.base_channels[s]) * elem_bytes(c);
}
// GroupNorm mode: statistics partials of one layer, (mean, M2) per (image, 128-pixel tile, 16-channel group)
size_t gn_part_bytes(const slim_config &c, int s, float r, int B) {
    if (c.norm != SLIM_NORM_GN || c.dtype != SLIM_BF16) return 0;
    const int H = seg_hw(c, s), tiles = H * H >= 128 ? H * H / 128 : 1;
    return round256(static_cast<size_t>(B) * tiles * (slim_act_channels(r, c.base_channels[s]) / 16 + 1) * 8);
}
// tile-flag counters of a segment's two flagged layer boundaries: one per M tile (<= 8 per image)
size_t tile_flag_bytes(const slim_config &c, int B) {
    return c.dtype == SLIM_BF16 ? round256(2 * static_cast<size_t>(B) * 8 * sizeof(uint32_t)) : 0;
}
// FP32 mode split-K (ConvF32Args::ksplit): K splits of segment s's layers -- every layer of a segment has the
// same output tiling -- from the tile count at max_batch (never B: the summation order is batch independent)
int f32_ksplit(const slim_config &c, int s, float r) {
    if (c.dtype != SLIM_FP32 || getenv("SLIM_F32_NO_SPLITK")) return 1;
    const int H = seg_hw(c, s), C = slim_act_channels(r, c.base_channels[s]);
    const long tiles = (static_cast<long>(c.max_batch) * H * H + 127) / 128 * ((C + 63) / 64);
    return tiles >= 148 ? 1 : static_cast<int>(std::min<long>(4, std::max<long>(1, 296 / tiles)));
}
size_t f32_part_bytes(const slim_config &c, int s, float r, int B) {
    const int ks = f32_ksplit(c, s, r);
    return ks > 1 ? round256((ks + 1) * act_bytes(c, s, r, B)) : 0;   // + the projection's slot
}
size_t seg_ws_bytes(const slim_config &c, int s, float r, int B) {
    return 3 * round256(act_bytes(c, s, r, B)) + gn_part_bytes(c, s, r, B) + tile_flag_bytes(c, B) +
           f32_part_bytes(c, s, r, B);
}

uint16_t f2bf(float f) {   // round-to-nearest-even (NaN kept NaN)
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x7FFFFFu)) return static_cast<uint16_t>((u >> 16) | 0x40);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}
float bf_round(float f) {
    uint32_t u = static_cast<uint32_t>(f2bf(f)) << 16;
    float r;
    std::memcpy(&r, &u, 4);
    return r;
}

#define CUDA_TRY(ctx, expr)                                                                            \
    do {                                                                                               \
        cudaError_t e__ = (expr);                                                                      \
        if (e__ != cudaSuccess) return fail((ctx), SLIM_ECUDA, "%s: %s", #expr, cudaGetErrorString(e__)); \
    } while (0)

// Brackets one kernel launch: counts it and, while profiling, records an event pair
// and the launch's algorithmic work.
struct LaunchProf {
    slim_ctx *ctx;
    cudaStream_t st;
    int idx = -1;
    LaunchProf(slim_ctx *c, cudaStream_t s) : ctx(c), st(s) {
        if (ctx->prof_on && 2 * (ctx->prof_rec.size() + 1) <= ctx->prof_ev.size()) {
            idx = static_cast<int>(ctx->prof_rec.size());
            cudaEventRecord(ctx->prof_ev[2 * idx], st);
        }
    }
    void done(int kind, int seg, int layer, float r_prev, float r, int B, double flops, double bytes) {
        ctx->launches++;
        if (idx >= 0) {
            cudaEventRecord(ctx->prof_ev[2 * idx + 1], st);
            slim_profile_record rec{kind, seg, layer, B, r_prev, r, flops, bytes, 0.f};
            ctx->prof_rec.push_back(rec);
        }
    }
};

void clear_graphs(slim_ctx *ctx) {
    std::lock_guard<std::mutex> g(ctx->graph_mu);
    for (auto &kv : ctx->graphs) cudaGraphExecDestroy(kv.second.exec);
    ctx->graphs.clear();
}

CUtensorMapSwizzle swizzle_for(int box_c) {   // box inner bytes = 2*box_c = the swizzle span
    return box_c == 16 ? CU_TENSOR_MAP_SWIZZLE_32B : (box_c == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B);
}

// Encoded tensor maps are cached by their full argument list (eager launches re-encode the same
// activation maps for every call on the same buffers; the cache takes that host cost off the
// launch path of the executors).
bool encode_map(slim_ctx *ctx, CUtensorMap *tm, const void *ptr, int rank, const cuuint64_t *dims,
                const cuuint64_t *strides, const cuuint32_t *box, const cuuint32_t *es, bool swizzle = true) {
    uint64_t key[1 + 1 + 5 + 4 + 5 + 5 + 1] = {};
    key[0] = reinterpret_cast<uintptr_t>(ptr);
    key[1] = static_cast<uint64_t>(rank);
    for (int i = 0; i < rank; ++i) {
        key[2 + i] = dims[i];
        key[11 + i] = box[i];
        key[16 + i] = es[i];
    }
    for (int i = 0; i + 1 < rank; ++i) key[7 + i] = strides[i];
    key[21] = swizzle;
    const std::string k(reinterpret_cast<const char *>(key), sizeof key);
    {
        std::lock_guard<std::mutex> g(ctx->tm_mu);
        auto it = ctx->tm_cache.find(k);
        if (it != ctx->tm_cache.end()) {
            *tm = it->second;
            return true;
        }
    }
    CUresult r = ctx->encode(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void *>(ptr), dims, strides, box,
                             es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             swizzle ? swizzle_for(static_cast<int>(box[0])) : CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    std::lock_guard<std::mutex> g(ctx->tm_mu);
    if (ctx->tm_cache.size() > 8192) ctx->tm_cache.clear();
    ctx->tm_cache.emplace(k, *tm);
    return true;
}

// Activation NHWC [B][H][W][C] bf16 as a 4-D map (C, W, H, B); box (box_c, bw, bh, bn), traversal
// stride es in H, W.  box_c = 16 | 32 | 64 channels selects SWIZZLE_32B | 64B | 128B.
bool encode_act(slim_ctx *ctx, CUtensorMap *tm, const void *ptr, int B, int H, int W, int C, int bw, int bh, int bn,
                int es, int box_c = kChunk) {
    cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)B};
    cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
    cuuint32_t box[4] = {(cuuint32_t)box_c, (cuuint32_t)bw, (cuuint32_t)bh, (cuuint32_t)bn};
    cuuint32_t est[4] = {1, (cuuint32_t)es, (cuuint32_t)es, 1};
    return encode_map(ctx, tm, ptr, 4, dims, strides, box, est);
}

// The same NHWC activation addressed as (C, W, N, H) -- the image index inside the row index --
// so that a box [box_c, W, bn, bh] lands in shared memory as (row, image, column) (halo kernel).
// es = 2: traversal stride 2 in W and H (box W*es x bh*es elements, every other one delivered).
bool encode_act_rowmajor(slim_ctx *ctx, CUtensorMap *tm, const void *ptr, int B, int H, int W, int C, int bn, int bh,
                         int box_c, int es = 1) {
    cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)B, (cuuint64_t)H};
    cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)H * W * C * 2, (cuuint64_t)W * C * 2};
    cuuint32_t box[4] = {(cuuint32_t)box_c, (cuuint32_t)W, (cuuint32_t)bn, (cuuint32_t)(bh * es)};
    cuuint32_t est[4] = {1, (cuuint32_t)es, 1, (cuuint32_t)es};
    return encode_map(ctx, tm, ptr, 4, dims, strides, box, est);
}

// channels per operand chunk: exact narrow boxes for 16 / 32 channels, else 64 (128-B rows)
int chunk_ch(int c) {
    static const bool wide = getenv("SLIM_WIDE_BOX") != nullptr;   // diagnostics: always 64-channel boxes
    return (!wide && (c == 16 || c == 32)) ? c : kChunk;
}

// Weights KRSC [Cout_full][k*k][Cin_full] bf16 as a 3-D map whose BOUNDS are the
// active prefix (c_in, k*k, c_out): the slice is selected by predication.
bool encode_w(slim_ctx *ctx, CUtensorMap *tm, const DevLayer &L, int c_in, int c_out, int n_tile, int box_c = 0) {
    const int kk = L.sh.k * L.sh.k;
    cuuint64_t dims[3] = {(cuuint64_t)c_in, (cuuint64_t)kk, (cuuint64_t)c_out};
    cuuint64_t strides[2] = {(cuuint64_t)L.sh.cin * 2, (cuuint64_t)kk * L.sh.cin * 2};
    cuuint32_t box[3] = {(cuuint32_t)(box_c ? box_c : chunk_ch(c_in)), 1, (cuuint32_t)n_tile};
    cuuint32_t est[3] = {1, 1, 1};
    return encode_map(ctx, tm, L.w, 3, dims, strides, box, est);
}

// N per CTA tile: the widest divisor of c_out that is a multiple of 16 and <= 256
// (the UMMA N limit), narrowed down to 64 while the grid would leave most SMs idle
// (small-M layers late in the network, SURVEY §7 "hard parts" #3).  When there are
// several N tiles each must be a multiple of 64 channels.
// Weights as a 3-D map (ci, co, tap) -- strides co: 9*Cin_full*2, tap: Cin_full*2 -- so a box
// [64, n_tile, taps] lands as `taps` consecutive K-major n_tile x 64 operand tiles.
bool encode_w_taps(slim_ctx *ctx, CUtensorMap *tm, const DevLayer &L, int c_in, int c_out, int n_tile, int taps,
                   int box_c) {
    cuuint64_t dims[3] = {(cuuint64_t)c_in, (cuuint64_t)c_out, 9};
    cuuint64_t strides[2] = {(cuuint64_t)9 * L.sh.cin * 2, (cuuint64_t)L.sh.cin * 2};
    cuuint32_t box[3] = {(cuuint32_t)box_c, (cuuint32_t)n_tile, (cuuint32_t)taps};
    cuuint32_t est[3] = {1, 1, 1};
    return encode_map(ctx, tm, L.w, 3, dims, strides, box, est);
}

int pick_n_tile(int c_out, int m_tiles = 1 << 30, int num_sms = 148) {
    int best = 0;
    for (int nt = 1; nt <= c_out / 16; ++nt) {
        if (c_out % nt || (c_out / nt) % 16) continue;
        const int n = c_out / nt;
        // several N tiles must each cover whole 64-channel staging chunks: the output
        // TMA box is 64 channels wide and would spill into the neighbour tile otherwise
        if (nt > 1 && n % 64) continue;
        if (n > 256) continue;
        if (best == 0) best = n;   // widest legal tile
        if (static_cast<long>(m_tiles) * nt * 10 >= static_cast<long>(num_sms) * 8 || n <= 64) {
            best = n;
            break;
        }
        best = n;
    }
    return best;
}

const CUtensorMap *weight_map(slim_ctx *ctx, DevLayer &L, int ri_in, int ri, int c_in, int c_out, int n_tile) {
    std::lock_guard<std::mutex> g(ctx->mu);
    if (!L.tm_ok[ri_in][ri][n_tile >> 4]) {
        if (!encode_w(ctx, &L.tm[ri_in][ri][n_tile >> 4], L, c_in, c_out, n_tile)) return nullptr;
        L.tm_ok[ri_in][ri][n_tile >> 4] = true;
    }
    return &L.tm[ri_in][ri][n_tile >> 4];
}

// One conv launch of a BasicBlock: out = epi(conv(x; L) [+ proj(xp; Lp)] [+ res]).
struct ConvCall {
    int seg = 0, layer = 0;                  // for profiling records
    DevLayer *L = nullptr;
    int ri_in = 0;                           // width index that sets c_in (r_prev for block-0 c1 of seg>0)
    const void *x = nullptr;
    int H = 0, W = 0, c_in = 0;
    DevLayer *Lp = nullptr;                  // 1x1 stride-2 projection (EPI_BN_PROJ_RELU)
    int ri_in_p = 0, layer_p = 0;
    const void *xp = nullptr;
    int Hp = 0, Wp = 0, c_in_p = 0;
    const void *res = nullptr;               // identity residual (EPI_BN_ADD_RELU)
    void *out = nullptr;
    float *pool_out = nullptr;               // fused global average pool (fp32 [B][c_out]) instead of `out`
    int epi = EPI_BN_RELU;
    float relu_lo = 0.f;                     // -inf: no ReLU (GroupNorm mode: raw pre-norm output)
    float2 *gn_part = nullptr;               // GroupNorm mode: where the conv may write statistics partials
    bool gn_fuse = false;                    // GroupNorm mode: normalise in the epilogue (halo, whole-image tiles)
    // tile-granular dependencies (halo path only, HaloArgs::flag_*); dry: fill *dry and launch nothing
    uint32_t *flag_in = nullptr, *flag_out = nullptr, *flag_zero = nullptr;
    int flag_in_target = 0, flag_zero_n = 0;
    HaloArgs *dry = nullptr;
    float *f32_part = nullptr;               // FP32 mode: split-K partials (workspace), nullptr = no split
    mutable bool gn_stats = false;           // set when the launched kernel wrote them (halo path)
    mutable int gn_tiles_per_img = 0;        // their tiling (partials per image per group)
};

// Algorithmic work: 2*MACs of the sliced conv(s); bytes = input(s),
// sliced weights, residual read once, output written once, folded BN vectors.
void conv_work(const slim_config &c, const ConvCall &cc, int ri, int B, int Ho, int Wo, double *flops,
               double *bytes) {
    const double eb = static_cast<double>(elem_bytes(c));
    const int k = cc.L->sh.k;
    const double c_out = slim_channels(c.widths[ri], cc.L->sh.cout);
    const double pix = static_cast<double>(B) * Ho * Wo;
    double f = 2.0 * pix * c_out * k * k * cc.c_in;
    double b = eb * (static_cast<double>(B) * cc.H * cc.W * cc.c_in + c_out * k * k * cc.c_in + pix * c_out) +
               8.0 * c_out;
    if (cc.epi == EPI_BN_ADD_RELU) b += eb * pix * c_out;
    if (cc.epi == EPI_BN_PROJ_RELU) {
        f += 2.0 * pix * c_out * cc.c_in_p;
        b += eb * (static_cast<double>(B) * cc.Hp * cc.Wp * cc.c_in_p + c_out * cc.c_in_p) + 8.0 * c_out;
    }
    *flops = f;
    *bytes = b;
}

// SM partitioning between concurrent width instances (slim_set_sm_share): the persistent grids of a
// width's kernels are capped at share * num_SMs, so the latency-bound kernels of several width
// instances running on their own streams occupy disjoint SM sets instead of each taking all SMs and
// serialising at kernel granularity.  SLIM_GRID_CAP="f0,f1,..." (per width index) overrides for A/B.
int grid_cap(const slim_ctx *ctx, int ri, int grid, int seg = -1) {
    static float env_frac[kMaxW] = {0};
    static const bool env_set = [] {
        const char *e = getenv("SLIM_GRID_CAP");
        if (!e || !*e) return false;
        for (int i = 0; i < kMaxW; ++i) env_frac[i] = 1.f;
        for (int i = 0; e && *e && i < kMaxW; ++i) {
            env_frac[i] = static_cast<float>(atof(e));
            e = strchr(e, ',');
            if (e) ++e;
        }
        return true;
    }();
    float f = env_set ? env_frac[ri] : ctx->sm_share[ri];
    static float seg_scale[4] = {1.f, 1.f, 1.f, 1.f};   // experiment: SLIM_SEG_CAP_SCALE="a,b,c,d"
    static const bool seg_parsed = [] {
        const char *e = getenv("SLIM_SEG_CAP_SCALE");
        for (int i = 0; e && *e && i < 4; ++i) {
            seg_scale[i] = static_cast<float>(atof(e));
            e = strchr(e, ',');
            if (e) ++e;
        }
        return true;
    }();
    (void)seg_parsed;
    if (seg >= 0 && seg < 4 && f < 1.f) f = f * seg_scale[seg] < 1.f ? f * seg_scale[seg] : 1.f;
    const int cap = static_cast<int>(f * ctx->num_sms + 0.5f);
    return (cap >= 1 && cap < grid) ? cap : grid;
}

// Stride-1 3x3 conv with one halo load per channel chunk (kernels_halo.cu).  Returns
// SLIM_EUNSUPPORTED (nothing launched) when the layer does not fit its constraints.
slim_status conv_halo_bf16(slim_ctx *ctx, cudaStream_t st, const ConvCall &cc, int ri, int B, bool allow_small = true) {
    static const bool disabled = getenv("SLIM_NO_HALO") != nullptr;
    const slim_config &c = ctx->cfg;
    DevLayer &L = *cc.L;
    static const bool no_proj = getenv("SLIM_HALO_NO_PROJ") != nullptr;
    static const bool no_s2 = getenv("SLIM_HALO_NO_S2") != nullptr;
    if (disabled || L.sh.k != 3 || (L.sh.stride != 1 && L.sh.stride != 2)) return SLIM_EUNSUPPORTED;
    const bool s2 = L.sh.stride == 2;   // stride-2 conv1 (parity planes): plain BN + ReLU epilogue only
    if (s2 && (no_s2 || cc.epi != EPI_BN_RELU || cc.pool_out || cc.H % 2 || cc.W % 2)) return SLIM_EUNSUPPORTED;
    const bool proj = cc.epi == EPI_BN_PROJ_RELU;
    if (proj && (no_proj || cc.Lp->sh.k != 1 || cc.Lp->sh.stride != 2 || cc.Hp != 2 * cc.H || cc.Wp != 2 * cc.W))
        return SLIM_EUNSUPPORTED;
    const int H = s2 ? cc.H / 2 : cc.H, W = s2 ? cc.W / 2 : cc.W;   // output size
    static const bool no_small = getenv("SLIM_HALO_NO_SMALL") != nullptr;   // A/B: small images via per-tap conv
    if (W > 32 || 32 % W) return SLIM_EUNSUPPORTED;
    const int c_out = slim_act_channels(c.widths[ri], L.sh.cout);
    HaloArgs a{};
    a.B = B;
    a.H = H;
    a.W = W;
    if (H * W >= kTileM) {   // a tile is kTileM/W whole rows of one image
        if (kTileM % W || H % (kTileM / W)) return SLIM_EUNSUPPORTED;
        a.tile_imgs = 1;
        a.rows = kTileM / W;
        a.tiles_per_img = H / a.rows;
        a.m_tiles = B * a.tiles_per_img;
    } else {                 // a tile is kTileM/(H*W) whole images
        if (no_small || kTileM % (H * W)) return SLIM_EUNSUPPORTED;
        a.tile_imgs = kTileM / (H * W);
        a.rows = H;
        a.tiles_per_img = 1;
        a.m_tiles = (B + a.tile_imgs - 1) / a.tile_imgs;
    }
    a.row_px = a.tile_imgs * W;
    // fused pool: one image row per TMEM lane quarter (the 4x4 images of the last segment)
    if (cc.pool_out && (a.tile_imgs == 1 || a.row_px != 32 || a.rows != 4 || proj)) return SLIM_EUNSUPPORTED;   // (no pool + projection variant)
    a.pool_out = cc.pool_out;
    a.relu_lo = cc.relu_lo;
    // N tile <= 128: three accumulators of it must fit the 512 TMEM columns
    // (128-channel layers: two N tiles of 64 keep two accumulator stages + the fused N=192 MMA,
    // measured faster than one tile of 128; 96 channels cannot split into 64-channel tiles)
    static const int halo_nmax_env = getenv("SLIM_HALO_NMAX") ? atoi(getenv("SLIM_HALO_NMAX")) : 0;
    const int halo_nmax = halo_nmax_env ? halo_nmax_env : (c_out % 64 == 0 && c_out > 64 ? 64 : 128);
    int nt = 1;
    for (;; ++nt) {
        if (nt > c_out / 16) return SLIM_EUNSUPPORTED;
        if (c_out % nt || (c_out / nt) % 16 || (nt > 1 && (c_out / nt) % 64)) continue;
        if (c_out / nt <= halo_nmax) break;
    }
    // too few tiles to fill the SMs (narrow late layers): narrower N tiles of 32 / 16 channels with
    // exact-width output boxes -- each CTA's serial latency chain (MMA, epilogue) shrinks with it
    static const bool no_fill = getenv("SLIM_HALO_NOFILL") != nullptr;
    bool narrow_out = false;
    // (experiment) SLIM_HALO_SPLITN=32: 32-channel N tiles for single-chunk layers -> more accumulator
    // stages / tile groups in flight per CTA
    static const int splitn = getenv("SLIM_HALO_SPLITN") ? atoi(getenv("SLIM_HALO_SPLITN")) : 0;
    if ((splitn == 32 || splitn == 16) && !cc.pool_out && cc.c_in <= kChunk && c_out / nt > splitn && c_out % splitn == 0) {
        nt = c_out / splitn;
        narrow_out = true;
    }
    // Widths whose channel count is not a multiple of 64 above 64 (r = 0.75: 96 at segment 1): one N
    // tile of 96 gives 3 x 96 accumulator columns, so only ONE accumulator stage fits TMEM and the MMA
    // of tile i+1 cannot overlap the epilogue of tile i.  Narrower N tiles with exact-width output boxes
    // restore 2-4 stages.  SLIM_HALO_SPLITW = 0 (off) | 32 | 48 (A/B).
    static const int splitw_env = getenv("SLIM_HALO_SPLITW") ? atoi(getenv("SLIM_HALO_SPLITW")) : 0;
    if (!narrow_out && nt == 1 && 3 * c_out > 256 && c_out % 64 && splitw_env > 0 && c_out % splitw_env == 0 &&
        splitw_env % 16 == 0) {
        nt = c_out / splitw_env;
        narrow_out = true;
    }
    // (the SMs to fill are this width's share when instances are partitioned, slim_set_sm_share)
    const int fill_sms = grid_cap(ctx, ri, ctx->num_sms, cc.seg);
    if (!no_fill && a.m_tiles * nt * 10 < fill_sms * 8 && !cc.pool_out)
        for (int n2 : {32, 16}) {
            if (n2 >= c_out / nt || c_out % n2 || a.m_tiles * (c_out / n2) > fill_sms) continue;   // one wave
            nt = c_out / n2;
            narrow_out = true;
            if (a.m_tiles * nt * 10 >= fill_sms * 8) break;
        }
    a.n_tile = c_out / nt;
    a.n_tiles = nt;
    a.c_out = c_out;
    a.c_in = cc.c_in;
    // compact variant for narrow layers (c_out <= 32, c_in <= 64; opt-in SLIM_HALO_SMALL=1): exact
    // 16/32-channel boxes, <= 256 TMEM columns and ~110 KB of smem so two CTAs share an SM.  Measured:
    // -13 % on seg 0 at r <= 0.5 for one width alone, but the concurrent 4-width step loses 4 %: a
    // compact CTA parked on an SM holds off the full-SM CTAs of the wide instances' kernels
    static const int small_env = getenv("SLIM_HALO_SMALL") ? atoi(getenv("SLIM_HALO_SMALL")) : 0;
    bool small = allow_small && small_env != 0 && c_out <= 32 && cc.c_in <= 64 && !cc.pool_out;
    // 64-channel boxes unless SLIM_HALO_NARROW or the compact variant (16/32-channel boxes)
    static const bool halo_narrow = getenv("SLIM_HALO_NARROW") != nullptr;
    auto hch = [&](int ch) { return (halo_narrow || small) ? chunk_ch(ch) : kChunk; };
    a.ck = proj ? kChunk : hch(cc.c_in);
    a.rbk = 2 * a.ck;
    a.n_chunks = (cc.c_in + a.ck - 1) / a.ck;
    // exact-width output boxes: the widest 64 / 32 / 16-channel box dividing the tile (a 48-channel tile
    // stores three 16-channel boxes: the staging rows must be a swizzle span of 32, 64 or 128 B)
    a.co_chunk = narrow_out ? (a.n_tile % 64 == 0 ? 64 : (a.n_tile % 32 == 0 ? 32 : 16)) : hch(a.n_tile);
    a.rbo = 2 * a.co_chunk;
    a.epi = cc.epi;
    a.scale = L.scale[ri];
    a.shift = L.shift[ri];
    if (cc.gn_fuse) {   // GroupNorm in the epilogue: the tile must hold whole images (their full statistics)
        // or, as an image pair, a CTA takes both M tiles of one image (segment 1)
        if ((a.tiles_per_img != 1 && a.tiles_per_img != 2) || small) return SLIM_EUNSUPPORTED;
        a.gn_pairs = a.tiles_per_img == 2 ? 1 : 0;
        a.gn_fuse = 1;
        a.gn_eps = c.bn_eps;
        a.scale = L.gn_gamma[ri];
        a.shift = L.gn_beta[ri];
        a.relu_lo = 0.f;
    }
    // kw taps share one MMA (N = k*n_tile <= 256, the three accumulators adjacent in TMEM, the
    // tap blocks of B adjacent in smem) unless SLIM_HALO_NOFUSE
    static const bool nofuse = getenv("SLIM_HALO_NOFUSE") != nullptr;
    a.kw_fuse = nofuse ? 1 : (3 * a.n_tile <= 256 ? 3 : (2 * a.n_tile <= 256 ? 2 : 1));
    // x3 (three kw-shifted boxes, one accumulator, no shuffles): an alternative for the epilogue-bound
    // single-chunk layers (seg 0); measured 15% slower there (3x A traffic, N=64 MMAs): SLIM_HALO_X3=1
    static const int x3_env = getenv("SLIM_HALO_X3") ? atoi(getenv("SLIM_HALO_X3")) : -1;
    // x2 (two boxes, two accumulators, 2/3 of the TMEM reads): SLIM_HALO_X3=2, measured 5% slower at seg 0
    const bool xbox_ok = !a.gn_fuse && !small && !s2 && !proj && !cc.pool_out && cc.c_in <= kChunk && nt == 1 && 9 * a.n_tile * 128 <= 100 * 1024 &&
                         2 * a.n_tile <= 256;   // (weights stationary)
    const int xmode = !xbox_ok ? 0 : (x3_env >= 0 ? x3_env : 0);   // both measured slower than kw accumulators
    const bool x3 = xmode == 1, x2 = xmode == 2;
    if (x3 || x2) {
        a.x3 = xmode;
        a.kw_fuse = 1;
        a.gn_part = nullptr;   // (the x3 / x2 epilogues do not compute GN statistics)
    }
    if (s2) {   // [acc_kw0 | acc_kw2 | acc_kw1] adjacent; kw 0 and 2 as one N = 2n MMA
        if (2 * a.n_tile > 256) return SLIM_EUNSUPPORTED;
        a.kw_fuse = 3;
        a.stride2 = 1;
    }
    a.acc_stride = a.kw_fuse > 1 ? a.n_tile : (a.n_tile + 31) / 32 * 32;
    a.stage_cols = (3 * a.acc_stride + (proj ? a.n_tile : 0) + 31) / 32 * 32;
    if (x3) a.stage_cols = (a.n_tile + 31) / 32 * 32;   // one accumulator
    if (x2) {                                            // [acc_m | acc_2] adjacent (one N = 2n MMA)
        a.acc_stride = a.n_tile;
        a.stage_cols = (2 * a.n_tile + 31) / 32 * 32;
    }
    // up to four accumulator stages (narrow layers): the MMA runs further ahead of the epilogue,
    // whose per-tile latency chain (not its work) bounds narrow widths
    static const int max_stages = getenv("SLIM_HALO_STAGES") ? atoi(getenv("SLIM_HALO_STAGES")) : 4;
    const int tmem_max = small ? 256 : 512;
    a.acc_stages = (4 * a.stage_cols <= tmem_max && max_stages >= 4) ? 4
                                                                      : (2 * a.stage_cols <= tmem_max && max_stages >= 2 ? 2 : 1);
    if (a.gn_pairs) {   // both tiles of an image resident: exactly two stages, one tile group
        if (2 * a.stage_cols > tmem_max) return SLIM_EUNSUPPORTED;
        a.acc_stages = 2;
    }
    if (a.stage_cols > tmem_max) small = false;   // (cannot happen for c_out <= 64)
    int cols = a.acc_stages * a.stage_cols, tc = 32;
    while (tc < cols) tc <<= 1;
    a.tmem_cols = tc;
    a.a_bytes = static_cast<uint32_t>(kTileM + 2 * a.row_px) * a.rbk;
    if (s2) a.a_bytes = 2u * static_cast<uint32_t>((a.rows + 1) * a.row_px) * a.rbk;   // odd-row pair (the larger)
    a.a_slot = (a.a_bytes + 1023u) & ~1023u;

    if (proj) {   // a projection chunk = 128 px x 64 ch + its n_tile x 64 weights in one slot
        if (a.ck != kChunk) return SLIM_EUNSUPPORTED;
        a.scale1 = a.gn_fuse ? cc.Lp->gn_gamma[ri] : cc.Lp->scale[ri];
        a.shift1 = a.gn_fuse ? cc.Lp->gn_beta[ri] : cc.Lp->shift[ri];
        a.c_in_p = cc.c_in_p;
        a.n_chunks_p = (cc.c_in_p + kChunk - 1) / kChunk;
        a.a_slot = std::max<uint32_t>(a.a_slot, 16384u + static_cast<uint32_t>(a.n_tile) * 128u);
    }
    a.n_out_chunks = static_cast<uint32_t>((a.n_tile + a.co_chunk - 1) / a.co_chunk);
    const size_t chunk = static_cast<size_t>(a.n_out_chunks) * 128 * a.rbo;
    static const bool one_group = getenv("SLIM_HALO_EPI1") != nullptr;
    a.epi_groups = (one_group || a.gn_pairs) ? 1 : a.acc_stages;
    if (small && a.epi_groups > 2) a.epi_groups = 2;   // 8 epilogue warps: one or two tile groups
    a.small = small ? 1 : 0;
    const bool two = small;
    const size_t budget = two ? 110 * 1024 : 226 * 1024;
    // GroupNorm statistics partials (GN mode, plain / stride-2 variants): smem for the per-quarter merge.
    // Opt-in (SLIM_GN_PART=1): measured slower than the separate GN reduction kernel -- the statistics
    // add ~22 % to the epilogue-bound conv (seg 0 r=1: 18.8 -> 23.0 us standalone) while the elementwise
    // apply costs the same launch as the reduction kernel it replaces (GN CFG2 step 663 k vs 716 k images/s,
    // tools/gpu_runs/r02_gnpart.sh); kept as the measured alternative.
    static const bool no_gn_part = getenv("SLIM_GN_PART") == nullptr || getenv("SLIM_GN_NO_PART") != nullptr;
    a.gn_part = (cc.gn_part && !no_gn_part && !proj && !cc.pool_out && !small && !a.x3 && !a.gn_fuse) ? cc.gn_part : nullptr;
    auto fixed0 = [&]() {
        return 1024 + chunk * a.epi_groups + (proj ? 16 : 8) * static_cast<size_t>(c_out) + 8 * kHaloBars + 16 +
               (a.gn_part ? static_cast<size_t>(a.epi_groups) * (a.n_tile / 16) * 4 * a.tile_imgs * 16 + 16 : 0) +
               (a.gn_fuse ? static_cast<size_t>(a.epi_groups) * (a.n_tile / 16) * 4 * a.tile_imgs * 16 * (proj ? 2 : 1) *
                                    (a.gn_pairs ? 2 : 1) + 16
                          : 0);
    };
    auto r1k = [](uint32_t x) { return (x + 1023u) & ~1023u; };
    const uint32_t all_w = r1k(static_cast<uint32_t>(a.n_chunks) * 9u * a.n_tile * a.rbk);
    // residual slots: a multiple of the tile groups (each slot serves one group, parity waits)
    a.res_slots = (cc.epi == EPI_BN_ADD_RELU) ? std::max(2, a.epi_groups) : 0;
    a.stationary = (nt == 1 && all_w <= (small ? 48u : 100u) * 1024) ? 1 : 0;
    if (a.stationary) {
        a.b_bytes = all_w;
        a.sb = 1;
    } else {
        a.b_bytes = r1k(3u * a.n_tile * a.rbk);
    }
    // 2-SM MMA (cta_group::2, kernels_halo.cu): a CTA pair on consecutive M tiles of one N tile, one
    // M = 256 MMA per k-step, each CTA holding half of every B stage -- the layer's weight bytes from L2
    // and into each SM halve (streamed-weight layers: segments 1-3 at the wide widths).  SLIM_HALO_PAIR=0
    // turns it off (A/B).
    // Default: on from B = 1024 (same-box CFG3 A/B: +3-6 % per chain at B >= 1024 for every width, mixed
    // at B = 256-512, -1.6 % in the B = 128 CFG2 step; bit-identical either way, so the choice may depend on B).
    // SLIM_HALO_PAIR: 0 = off, 1 = every eligible layer, 2 = the stride-2 convs only.
    static const int pair_env = getenv("SLIM_HALO_PAIR") ? atoi(getenv("SLIM_HALO_PAIR")) : -1;
    // (128-channel layers only at segment 1: at segments 2-3 (r = 0.25 / 0.5) they measured slower)
    const int pair_mode = pair_env >= 0 ? pair_env : (B >= 1024 && (c_out >= 192 || cc.seg == 1) ? 1 : 0);
    const bool wide_boxes = a.ck == kChunk && a.co_chunk == kChunk;   // (the cluster variants are compiled for these)
    const bool pair = pair_mode != 0 && (pair_mode != 2 || s2) && !a.gn_fuse && wide_boxes && !a.stationary && !small && !a.x3 &&
                      a.kw_fuse == 3 && a.m_tiles % 2 == 0 &&
                      a.n_tile % 16 == 0 && !a.gn_part &&
                      grid_cap(ctx, ri, std::min(ctx->num_sms, a.m_tiles * a.n_tiles), cc.seg) >= 2;
    if (pair) {
        a.pair = 1;
        a.b_bytes = r1k(3u * (a.n_tile / 2) * a.rbk);
    }
    // fit: A slots 2..4, B slots 2..4 (streaming), residual slots 2 -> 1 if tight
    for (;;) {
        const size_t res = chunk * a.res_slots;
        size_t left = budget - fixed0() - res;
        if (a.stationary) {
            if (left < a.b_bytes + 2 * a.a_slot) {
                if (a.epi_groups > 1) {   // fewer tile groups (stages stay: a multiple of the groups)
                    a.epi_groups >>= 1;
                    if (a.res_slots) a.res_slots = std::max(2, a.epi_groups);
                    continue;
                }
                if (a.res_slots == 2) { a.res_slots = 1; continue; }
                return small ? conv_halo_bf16(ctx, st, cc, ri, B, false) : SLIM_EUNSUPPORTED;
            }
            left -= a.b_bytes;
            a.sa = static_cast<int>(left / a.a_slot);
            a.sa = a.sa > 4 ? 4 : a.sa;
        } else {
            if (left < 2 * a.a_slot + 2 * a.b_bytes) {
                if (a.epi_groups > 1) {   // fewer tile groups (stages stay: a multiple of the groups)
                    a.epi_groups >>= 1;
                    if (a.res_slots) a.res_slots = std::max(2, a.epi_groups);
                    continue;
                }
                if (a.res_slots == 2) { a.res_slots = 1; continue; }
                return small ? conv_halo_bf16(ctx, st, cc, ri, B, false) : SLIM_EUNSUPPORTED;
            }
            a.sa = 2;
            left -= 2 * a.a_slot;
            a.sb = static_cast<int>(left / a.b_bytes);
            const int sb_max = a.pair ? kMaxSB : 4;   // pair: half-size stages, twice as many in flight
            a.sb = a.sb > sb_max ? sb_max : a.sb;
            if (a.sb >= 4 && left - a.sb * a.b_bytes >= a.a_slot) a.sa = 3;
        }
        break;
    }
    if (a.res_slots == 0) a.res_slots = 1;   // unused without a residual
    a.flag_in = cc.flag_in;
    a.flag_in_target = cc.flag_in_target;
    a.flag_out = cc.pool_out ? nullptr : cc.flag_out;
    a.flag_zero = cc.flag_zero;
    a.flag_zero_n = cc.flag_zero_n;
    if (cc.dry) {   // shape-only query: would the halo kernel take this layer, and how is it tiled
        *cc.dry = a;
        return SLIM_OK;
    }
    static const int conv_debug = getenv("SLIM_CONV_DEBUG") ? atoi(getenv("SLIM_CONV_DEBUG")) : 0;
    a.debug = conv_debug;
    a.trace = ctx->trace;

    CUtensorMap tA, tRes, tOut, tA1, tB1, tBs;
    if (!s2 && !encode_act_rowmajor(ctx, &tA, cc.x, B, H, W, cc.c_in, a.tile_imgs, a.rows + 2, a.ck))
        return fail(ctx, SLIM_ECUDA, "cuTensorMapEncodeTiled(halo A) failed");
    if (s2 && (!encode_act_rowmajor(ctx, &tA, cc.x, B, cc.H, cc.W, cc.c_in, a.tile_imgs, a.rows, a.ck, 2) ||
               !encode_act_rowmajor(ctx, &tA1, cc.x, B, cc.H, cc.W, cc.c_in, a.tile_imgs, a.rows + 1, a.ck, 2)))
        return fail(ctx, SLIM_ECUDA, "cuTensorMapEncodeTiled(halo s2 A) failed");
    const int taps = a.stationary ? 9 : 3;
    const CUtensorMap *tB;
    if (s2) {   // one-tap boxes (the kernel reorders kw per kh); c_in = c(r_prev): not cached per r
        if (!encode_w_taps(ctx, &tBs, L, cc.c_in, c_out, a.n_tile, 1, a.ck))
            return fail(ctx, SLIM_ECUDA, "cuTensorMapEncodeTiled(halo s2 W) failed");
        tB = &tBs;
    } else {
        std::lock_guard<std::mutex> g(ctx->mu);
        bool &ok = L.tmh_ok[ri][a.n_tile / 16 - 1][a.stationary];
        CUtensorMap &m = L.tmh[ri][a.n_tile / 16 - 1][a.stationary];
        if (!ok) {
            if (!encode_w_taps(ctx, &m, L, cc.c_in, c_out, a.n_tile, taps, a.ck))
                return fail(ctx, SLIM_ECUDA, "cuTensorMapEncodeTiled(halo W) failed");
            ok = true;
        }
        tB = &m;
    }
    if (!encode_act_rowmajor(ctx, &tOut, cc.pool_out ? cc.x : cc.out, B, H, W, c_out, a.tile_imgs, a.rows, a.co_chunk))
        return fail(ctx, SLIM_ECUDA, "cuTensorMapEncodeTiled(halo out) failed");
    tRes = tOut;
    if (cc.epi == EPI_BN_ADD_RELU &&
        !encode_act_rowmajor(ctx, &tRes, cc.res, B, H, W, c_out, a.tile_imgs, a.rows, a.co_chunk))
        return fail(ctx, SLIM_ECUDA, "cuTensorMapEncodeTiled(halo res) failed");
    const int total = a.m_tiles * a.n_tiles;
    int grid = ctx->num_sms * (two ? 2 : 1);
    if (grid > total) grid = total;
    if (a.gn_pairs && grid > total / 2) grid = total / 2;   // a CTA's tiles come in image pairs
    grid = grid_cap(ctx, ri, grid, cc.seg);
    if (a.pair) grid -= grid % 2;   // (>= 2: checked with the pair decision)
    // tile order: SLIM_HALO_NFAST = 1 N-fastest, 0 M-fastest, unset = auto (see below)
    static const int nfast_env = getenv("SLIM_HALO_NFAST") ? atoi(getenv("SLIM_HALO_NFAST")) : -1;
    // auto: N-fastest once the layer's input no longer fits L2 (126 MB): then the M-fastest order streams the
    // input from DRAM once per N tile (B = 4096: r = 1 chain 4.95 -> 4.60 ms, r = 0.75 3.55 -> 3.44 ms), while
    // with an L2-resident input it keeps each weight tile hot (B = 1024: M-fastest 5 % faster); bit-identical
    const double in_bytes = 2.0 * B * cc.H * cc.W * cc.c_in;
    a.nfast = (a.n_tiles > 1 && (nfast_env == 1 || (nfast_env < 0 && in_bytes > 96e6))) ? 1 : 0;
    // streamed weights: clusters of bmc CTAs on consecutive M tiles of one N tile share each B stage
    // (TMA multicast) -- the weight bytes one launch pulls from L2 drop by bmc.  Opt-in (SLIM_HALO_BMC=2|4):
    // bit-identical, but measured no faster (B=1024 r=1 seg 2/3 convs 84/80 us either way; B=128 chains
    // +4 %, bmc 4 up to 2x slower: the cluster's CTAs advance in lock step, profiles/r02_bmc_multicast.txt),
    // so the L2->SM weight stream is not what bounds these convs
    static const int bmc_env = getenv("SLIM_HALO_BMC") ? atoi(getenv("SLIM_HALO_BMC")) : 1;
    a.bmc = 1;
    CUtensorMap tBh = tA;
    if (a.pair) {
        if (!encode_w_taps(ctx, &tBh, L, cc.c_in, c_out, a.n_tile / 2, s2 ? 1 : 3, a.ck))
            return fail(ctx, SLIM_ECUDA, "cuTensorMapEncodeTiled(halo W pair half) failed");
    } else if ((bmc_env == 2 || bmc_env == 4) && wide_boxes && !a.stationary && !small && !a.x3 && a.m_tiles % bmc_env == 0 &&
        (a.n_tile / bmc_env) % 8 == 0 && grid >= bmc_env) {
        if (!encode_w_taps(ctx, &tBh, L, cc.c_in, c_out, a.n_tile / bmc_env, 1, a.ck))
            return fail(ctx, SLIM_ECUDA, "cuTensorMapEncodeTiled(halo W share) failed");
        a.bmc = bmc_env;
        a.nfast = 0;   // (the multicast clusters take M-consecutive tiles of one N tile)
        grid -= grid % bmc_env;
    }
    double flops, bytes;
    conv_work(c, cc, ri, B, H, W, &flops, &bytes);
    if (ctx->trace) cudaMemsetAsync(ctx->trace, 0, 3584 * sizeof(unsigned long long), st);   // diagnostics (stem: 3584..)
    LaunchProf prof(ctx, st);
    if (!s2) tA1 = tA;
    tB1 = tA;
    if (proj) {
        if (!encode_act_rowmajor(ctx, &tA1, cc.xp, B, cc.Hp, cc.Wp, cc.c_in_p, a.tile_imgs, a.rows, kChunk, 2))
            return fail(ctx, SLIM_ECUDA, "cuTensorMapEncodeTiled(halo proj A) failed");
        if (!encode_w(ctx, &tB1, *cc.Lp, cc.c_in_p, c_out, a.pair ? a.n_tile / 2 : a.n_tile, kChunk))
            return fail(ctx, SLIM_ECUDA, "cuTensorMapEncodeTiled(halo proj W) failed");
    }
    cudaError_t e = launch_conv_halo(a, tA, *tB, tRes, tOut, tA1, tB1, tBh, grid, st, ctx->pdl && !ctx->prof_on);
    prof.done(SLIM_K_CONV_UMMA, cc.seg, cc.layer, c.widths[cc.ri_in], c.widths[ri], B, flops, bytes);
    if (e != cudaSuccess)
        return fail(ctx, SLIM_ECUDA, "conv_halo launch (grid %d, smem %zu): %s", grid, conv_halo_smem_bytes(a),
                    cudaGetErrorString(e));
    if (a.gn_part && !a.x3) {
        cc.gn_stats = true;
        cc.gn_tiles_per_img = a.tiles_per_img;
    }
    return SLIM_OK;
}

// Split-K over a cluster (kernels_splitk.cu) for layers whose M is too small to fill the SMs with
// wide tiles.  The split count depends only on the layer shape and the context's max_batch (never
// on B), so a layer's fp32 summation order -- and its output bits -- are batch independent.
// Returns SLIM_EUNSUPPORTED (nothing launched) when the layer does not qualify.
slim_status conv_splitk_bf16(slim_ctx *ctx, cudaStream_t st, const ConvCall &cc, int ri, int B) {
    static const bool disabled = getenv("SLIM_NO_SPLITK") != nullptr;
    // clusters of 8 measured far slower than 4 (cluster scheduling): 4 unless SLIM_SPLITK_MAX
    static const int ks_max = getenv("SLIM_SPLITK_MAX") ? atoi(getenv("SLIM_SPLITK_MAX")) : 4;
    const slim_config &c = ctx->cfg;
    DevLayer &L = *cc.L;
    if (disabled) return SLIM_EUNSUPPORTED;
    const int k = L.sh.k, s = L.sh.stride, pad = k / 2;
    const int Ho = (cc.H + 2 * pad - k) / s + 1, Wo = (cc.W + 2 * pad - k) / s + 1;
    const int c_out = slim_act_channels(c.widths[ri], L.sh.cout);
    const int P = Ho * Wo;
    SplitArgs a{};
    a.B = B;
    a.Ho = Ho;
    a.Wo = Wo;
    int m_ref;
    if (P >= kTileM) {
        if (P % kTileM || kTileM % Wo) return SLIM_EUNSUPPORTED;
        a.tile_imgs = 1;
        a.tile_rows = kTileM / Wo;
        a.tiles_per_img = Ho / a.tile_rows;
        a.m_tiles = B * a.tiles_per_img;
        m_ref = c.max_batch * a.tiles_per_img;
    } else {
        if (kTileM % P) return SLIM_EUNSUPPORTED;
        a.tile_imgs = kTileM / P;
        a.tile_rows = Ho;
        a.tiles_per_img = 1;
        a.m_tiles = (B + a.tile_imgs - 1) / a.tile_imgs;
        m_ref = (c.max_batch + a.tile_imgs - 1) / a.tile_imgs;
    }
    a.n_parts = (cc.epi == EPI_BN_PROJ_RELU) ? 2 : 1;
    // widest N tile: a divisor of c_out, multiple of 16, <= 256, both parts' accumulators in TMEM
    int nt = 0;
    for (int d = 256; d >= 16; d -= 16)
        if (c_out % d == 0 && a.n_parts * d <= 512) {
            nt = d;
            break;
        }
    if (!nt) return SLIM_EUNSUPPORTED;
    a.n_tile = nt;
    a.c_out = c_out;
    const int n_tiles = c_out / nt;
    a.part[0] = GemmPart{k, s, pad, cc.c_in, kChunk, 128, (cc.c_in + kChunk - 1) / kChunk, 0};
    a.part[0].n_kblocks = k * k * a.part[0].n_chunks;
    if (a.n_parts == 2) {
        a.part[1] = GemmPart{cc.Lp->sh.k, cc.Lp->sh.stride, 0, cc.c_in_p, kChunk, 128, (cc.c_in_p + kChunk - 1) / kChunk, 0};
        a.part[1].n_kblocks = a.part[1].n_chunks;
    }
    const int G = a.part[0].n_kblocks + (a.n_parts == 2 ? a.part[1].n_kblocks : 0);
    a.epi = cc.epi;
    a.scale0 = L.scale[ri];
    a.shift0 = L.shift[ri];
    if (a.n_parts == 2) {
        a.scale1 = cc.Lp->scale[ri];
        a.shift1 = cc.Lp->shift[ri];
    }
    a.pool_out = cc.pool_out;
    a.relu_lo = cc.relu_lo;
    if (a.pool_out && (P > 32 || 32 % P || a.tile_imgs == 1)) return SLIM_EUNSUPPORTED;
    a.stage_bytes = 16384u + static_cast<uint32_t>(nt) * 128u;
    int tc = 32;
    while (tc < a.n_parts * nt) tc <<= 1;
    a.tmem_cols = tc;
    // Split count from a cycle model at B = max_batch (so the choice -- and the fp32 summation
    // order -- never depends on B).  Measured on B200 (tools/layer_times.py): these
    // layers are bound by L2->SM operand traffic at ~32 B/cycle per SM when all SMs stream, so a
    // k-block costs max(its A+B bytes / 32, 4 UMMAs of N), times
    // the number of waves.  A split adds ~4000 + 1000*ks cycles (cluster launch, two cluster barriers,
    // the reduction epilogue after the last MMA) and the DSMEM push at ~16 B/cycle.
    auto cyc = [](double n) { return std::max(36.0 + n / 4.0, n / 2.0); };
    auto blk = [&](double n) { return std::max((16384.0 + n * 128.0) / 32.0, 4.0 * cyc(n)); };
    const int sms = ctx->num_sms;
    auto waves = [&](long ctas) { return static_cast<double>((ctas + sms - 1) / sms); };
    double best_cost;
    {
        const int n_ns = pick_n_tile(c_out, m_ref, sms);
        best_cost = waves(static_cast<long>(m_ref) * (c_out / n_ns)) * G * blk(n_ns);
    }
    static const bool force = getenv("SLIM_SPLITK_FORCE") != nullptr;   // tests: exercise the kernel
    if (force) best_cost = 1e300;
    int best_ks = 0;
    for (int ks = 2; ks <= std::min(8, ks_max); ++ks) {
        if (nt % ks || (nt / ks) % 16 || G < ks) continue;
        const double cost = waves(static_cast<long>(m_ref) * n_tiles * ks) *
                            (std::ceil(static_cast<double>(G) / ks) * blk(nt) + 4000.0 + 1000.0 * ks +
                             (ks - 1) * a.n_parts * 128.0 * (nt / ks) * 4.0 / 16.0);
        if (cost < best_cost) {
            best_cost = cost;
            best_ks = ks;
        }
    }
    if (getenv("SLIM_DEBUG"))
        fprintf(stderr, "[slim] splitk seg%d L%d c_in %d c_out %d G %d m_ref %d: ks %d\n", cc.seg, cc.layer, cc.c_in,
                c_out, G, m_ref, best_ks);
    bool fits = false;
    for (int ks = best_ks; ks >= 2 && !fits; --ks) {
        if (nt % ks || (nt / ks) % 16 || G < ks) continue;
        a.ks = ks;
        a.w_o = nt / ks;
        a.co_chunk = a.w_o % 64 == 0 ? 64 : (a.w_o % 32 == 0 ? 32 : 16);
        a.rbo = 2 * a.co_chunk;
        a.n_out_chunks = static_cast<uint32_t>(a.w_o / a.co_chunk);
        const size_t slice = static_cast<size_t>(a.n_out_chunks) * 128 * a.rbo;
        const size_t fixed = 1024 + slice * (cc.epi == EPI_BN_ADD_RELU ? 2 : 1) + 16 * static_cast<size_t>(a.w_o) +
                             8 * (2 * 8 + 2) + 16;
        int stages = static_cast<int>((226 * 1024 - fixed) / a.stage_bytes);
        if (stages > 8) stages = 8;
        a.n_stages = stages;
        fits = stages >= 2 && static_cast<size_t>(stages) * a.stage_bytes >= conv_splitk_recv_bytes(a);
    }
    if (!fits) return SLIM_EUNSUPPORTED;
    static const int nprod = getenv("SLIM_NPROD") ? atoi(getenv("SLIM_NPROD")) : 3;
    a.n_prod = nprod < 1 ? 1 : (nprod > 3 ? 3 : nprod);
    if (a.n_prod > a.n_stages) a.n_prod = a.n_stages;

    CUtensorMap tA0, tA1, tRes, tOut;
    if (!encode_act(ctx, &tA0, cc.x, B, cc.H, cc.W, cc.c_in, s * Wo, s * a.tile_rows, a.tile_imgs, s, kChunk))
        return fail(ctx, SLIM_ECUDA, "cuTensorMapEncodeTiled(split A) failed");
    const CUtensorMap *tB0, *tB1;
    {
        std::lock_guard<std::mutex> g(ctx->mu);
        if (!L.tms_ok[cc.ri_in][ri]) {
            if (!encode_w(ctx, &L.tms[cc.ri_in][ri], L, cc.c_in, c_out, nt, kChunk))
                return fail(ctx, SLIM_ECUDA, "cuTensorMapEncodeTiled(split W) failed");
            L.tms_ok[cc.ri_in][ri] = true;
        }
        tB0 = tB1 = &L.tms[cc.ri_in][ri];
        if (a.n_parts == 2) {
            DevLayer &Lp = *cc.Lp;
            if (!Lp.tms_ok[cc.ri_in_p][ri]) {
                if (!encode_w(ctx, &Lp.tms[cc.ri_in_p][ri], Lp, cc.c_in_p, c_out, nt, kChunk))
                    return fail(ctx, SLIM_ECUDA, "cuTensorMapEncodeTiled(split W1) failed");
                Lp.tms_ok[cc.ri_in_p][ri] = true;
            }
            tB1 = &Lp.tms[cc.ri_in_p][ri];
        }
    }
    tA1 = tA0;
    if (a.n_parts == 2) {
        const int sp = cc.Lp->sh.stride;
        if (!encode_act(ctx, &tA1, cc.xp, B, cc.Hp, cc.Wp, cc.c_in_p, sp * Wo, sp * a.tile_rows, a.tile_imgs, sp,
                        kChunk))
            return fail(ctx, SLIM_ECUDA, "cuTensorMapEncodeTiled(split A1) failed");
    }
    if (!encode_act(ctx, &tOut, cc.pool_out ? cc.x : cc.out, B, Ho, Wo, c_out, Wo, a.tile_rows, a.tile_imgs, 1,
                    a.co_chunk))
        return fail(ctx, SLIM_ECUDA, "cuTensorMapEncodeTiled(split out) failed");
    tRes = tOut;
    if (cc.epi == EPI_BN_ADD_RELU &&
        !encode_act(ctx, &tRes, cc.res, B, Ho, Wo, c_out, Wo, a.tile_rows, a.tile_imgs, 1, a.co_chunk))
        return fail(ctx, SLIM_ECUDA, "cuTensorMapEncodeTiled(split res) failed");
    const int grid = a.m_tiles * n_tiles * a.ks;
    double flops, bytes;
    conv_work(c, cc, ri, B, Ho, Wo, &flops, &bytes);
    LaunchProf prof(ctx, st);
    cudaError_t e = launch_conv_splitk(a, tA0, *tB0, tA1, *tB1, tRes, tOut, grid, st, ctx->pdl && !ctx->prof_on);
    prof.done(SLIM_K_CONV_UMMA, cc.seg, cc.layer, c.widths[cc.ri_in], c.widths[ri], B, flops, bytes);
    if (e != cudaSuccess)
        return fail(ctx, SLIM_ECUDA, "conv_splitk launch (grid %d, ks %d, n_tile %d, smem %zu, stages %d): %s", grid,
                    a.ks, nt, conv_splitk_smem_bytes(a), a.n_stages, cudaGetErrorString(e));
    return SLIM_OK;
}

slim_status conv_bf16(slim_ctx *ctx, cudaStream_t st, const ConvCall &cc, int ri, int B) {
    {
        const slim_status hs = conv_halo_bf16(ctx, st, cc, ri, B);
        if (hs != SLIM_EUNSUPPORTED) return hs;
        const slim_status ss = conv_splitk_bf16(ctx, st, cc, ri, B);
        if (ss != SLIM_EUNSUPPORTED) return ss;
    }
    const slim_config &c = ctx->cfg;
    DevLayer &L = *cc.L;
    const int k = L.sh.k, s = L.sh.stride, pad = k / 2;
    const int Ho = (cc.H + 2 * pad - k) / s + 1, Wo = (cc.W + 2 * pad - k) / s + 1;
    const int c_out = slim_act_channels(c.widths[ri], L.sh.cout);
    ConvArgs a{};
    a.B = B;
    a.Ho = Ho;
    a.Wo = Wo;
    const int P = Ho * Wo;
    if (P >= kTileM) {
        if (P % kTileM || kTileM % Wo) return fail(ctx, SLIM_EUNSUPPORTED, "conv: output %dx%d not tileable", Ho, Wo);
        a.tile_imgs = 1;
        a.tile_rows = kTileM / Wo;
        a.tiles_per_img = Ho / a.tile_rows;
        a.m_tiles = B * a.tiles_per_img;
    } else {
        if (kTileM % P) return fail(ctx, SLIM_EUNSUPPORTED, "conv: output %dx%d not tileable", Ho, Wo);
        a.tile_imgs = kTileM / P;
        a.tile_rows = Ho;
        a.tiles_per_img = 1;
        a.m_tiles = (B + a.tile_imgs - 1) / a.tile_imgs;
    }
    a.n_tile = pick_n_tile(c_out, a.m_tiles, ctx->num_sms);
    // shared memory must hold >= 2 pipeline stages next to the staging tile, the residual
    // ring and the BN vectors: narrow the N tile (to a smaller 64-multiple) until it does
    for (;;) {
        const int coc = chunk_ch(a.n_tile);
        const uint32_t nch = static_cast<uint32_t>((a.n_tile + coc - 1) / coc);
        const size_t chk = static_cast<size_t>(nch) * 128 * 2 * coc;
        const int nres = cc.epi == EPI_BN_ADD_RELU ? (nch <= 2 ? 2 : 1) : 0;
        const size_t need = 1024 + chk * (1 + nres) + 16 * static_cast<size_t>(c_out) + 8 * (2 * kMaxStages + 8) + 16 +
                            2 * (kTileABytes + static_cast<size_t>(a.n_tile) * 128);
        if (need <= 226 * 1024) break;
        int nt2 = c_out / a.n_tile + 1;
        while (nt2 <= c_out / 64 && (c_out % nt2 || (c_out / nt2) % 64)) ++nt2;
        if (nt2 > c_out / 64) return fail(ctx, SLIM_EUNSUPPORTED, "conv: no N tile fits shared memory");
        a.n_tile = c_out / nt2;
    }
    a.n_tiles = c_out / a.n_tile;
    a.c_out = c_out;
    a.n_parts = (cc.epi == EPI_BN_PROJ_RELU) ? 2 : 1;
    {
        const int ck0 = chunk_ch(cc.c_in);
        a.part[0] = GemmPart{k, s, pad, cc.c_in, ck0, 2 * ck0, (cc.c_in + ck0 - 1) / ck0, 0};
    }
    a.part[0].n_kblocks = k * k * a.part[0].n_chunks;
    if (a.n_parts == 2) {
        const int ck1 = chunk_ch(cc.c_in_p);
        a.part[1] = GemmPart{cc.Lp->sh.k, cc.Lp->sh.stride, 0, cc.c_in_p, ck1, 2 * ck1, (cc.c_in_p + ck1 - 1) / ck1, 0};
        a.part[1].n_kblocks = a.part[1].n_chunks;
    }
    a.epi = cc.epi;
    a.scale0 = L.scale[ri];
    a.shift0 = L.shift[ri];
    if (a.n_parts == 2) {
        a.scale1 = cc.Lp->scale[ri];
        a.shift1 = cc.Lp->shift[ri];
    }
    static const int conv_debug = getenv("SLIM_CONV_DEBUG") ? atoi(getenv("SLIM_CONV_DEBUG")) : 0;
    a.debug = conv_debug;
    a.trace = ctx->trace;   // diagnostics only
    a.acc_stride = (a.n_tile + 31) / 32 * 32;
    a.acc_stages = 512 / (a.n_parts * a.acc_stride) >= 2 ? 2 : 1;
    int cols = a.acc_stages * a.n_parts * a.acc_stride, tc = 32;
    while (tc < cols) tc <<= 1;
    a.tmem_cols = tc;
    {
        const int rbk = a.n_parts == 2 ? (a.part[0].rbk > a.part[1].rbk ? a.part[0].rbk : a.part[1].rbk) : a.part[0].rbk;
        a.a_tile_bytes = static_cast<uint32_t>(kTileM) * rbk;
        a.stage_b_bytes = (static_cast<uint32_t>(a.n_tile) * rbk + 1023u) & ~1023u;
    }
    a.co_chunk = chunk_ch(a.n_tile);
    a.rbo = 2 * a.co_chunk;
    a.n_out_chunks = static_cast<uint32_t>((a.n_tile + a.co_chunk - 1) / a.co_chunk);
    a.res_slots = a.n_out_chunks <= 2 ? 2 : 1;
    a.pool_out = cc.pool_out;
    a.relu_lo = cc.relu_lo;
    if (a.pool_out && (P > 32 || 32 % P || (a.tile_imgs == 1 && P != kTileM)))
        return fail(ctx, SLIM_EUNSUPPORTED, "fused pool needs Ho*Wo dividing 32");
    // pipeline depth: two CTAs per SM for very narrow tiles, one otherwise; 2..8 stages
    // in what the staging / residual ring / BN vectors leave
    const bool two = a.n_tile <= 32;
    const size_t budget = two ? 113 * 1024 : 226 * 1024;
    const size_t chunk = static_cast<size_t>(a.n_out_chunks) * 128 * a.rbo;
    const size_t fixed = 1024 + chunk * (1 + (cc.epi == EPI_BN_ADD_RELU ? a.res_slots : 0)) +
                         16 * static_cast<size_t>(c_out) + 8 * (2 * kMaxStages + 8) + 16;
    int stages = static_cast<int>((budget - fixed) / (a.a_tile_bytes + a.stage_b_bytes));
    a.n_stages = stages < 2 ? 2 : (stages > kMaxStages ? kMaxStages : stages);

    // TMA issue is bounded per issuing thread (~1 instruction per ~500 cycles), so up to four
    // producer warps take turns by k-block
    static const int nprod = getenv("SLIM_NPROD") ? atoi(getenv("SLIM_NPROD")) : 3;
    a.n_prod = nprod < 1 ? 1 : (nprod > 4 ? 4 : nprod);
    // producers take k-blocks round-robin and each checks its stage's empty barrier by parity:
    // with n_stages >= n_prod a producer is never two phases ahead on a stage (no parity aliasing)
    if (a.n_prod > a.n_stages) a.n_prod = a.n_stages;
    const int box_rows = a.tile_rows, box_imgs = a.tile_imgs;
    CUtensorMap tA0, tA1, tRes, tOut;
    if (!encode_act(ctx, &tA0, cc.x, B, cc.H, cc.W, cc.c_in, s * Wo, s * box_rows, box_imgs, s, a.part[0].ck))
        return fail(ctx, SLIM_ECUDA, "cuTensorMapEncodeTiled(A) failed");
    const CUtensorMap *tB0 = weight_map(ctx, L, cc.ri_in, ri, cc.c_in, c_out, a.n_tile);
    const CUtensorMap *tB1 = tB0;
    if (!tB0) return fail(ctx, SLIM_ECUDA, "cuTensorMapEncodeTiled(W) failed");
    tA1 = tA0;
    if (a.n_parts == 2) {
        const int sp = cc.Lp->sh.stride;
        if (!encode_act(ctx, &tA1, cc.xp, B, cc.Hp, cc.Wp, cc.c_in_p, sp * Wo, sp * box_rows, box_imgs, sp,
                        a.part[1].ck))
            return fail(ctx, SLIM_ECUDA, "cuTensorMapEncodeTiled(A1) failed");
        tB1 = weight_map(ctx, *cc.Lp, cc.ri_in_p, ri, cc.c_in_p, c_out, a.n_tile);
        if (!tB1) return fail(ctx, SLIM_ECUDA, "cuTensorMapEncodeTiled(W1) failed");
    }
    if (!encode_act(ctx, &tOut, cc.pool_out ? cc.x : cc.out, B, Ho, Wo, c_out, Wo, a.tile_rows, a.tile_imgs, 1,
                    a.co_chunk))
        return fail(ctx, SLIM_ECUDA, "cuTensorMapEncodeTiled(out) failed");
    tRes = tOut;
    if (cc.epi == EPI_BN_ADD_RELU &&
        !encode_act(ctx, &tRes, cc.res, B, Ho, Wo, c_out, Wo, a.tile_rows, a.tile_imgs, 1, a.co_chunk))
        return fail(ctx, SLIM_ECUDA, "cuTensorMapEncodeTiled(res) failed");

    const size_t smem = conv_umma_smem_bytes(a);
    const int per_sm = conv_umma_max_ctas_per_sm(smem);
    const int total = a.m_tiles * a.n_tiles;
    int grid = ctx->num_sms * per_sm;
    if (grid > total) grid = total;
    grid = grid_cap(ctx, ri, grid, cc.seg);
    // A-tile multicast: a cluster of mc CTAs (<= 8, dividing n_tiles) shares each M tile
    static const bool no_mc = getenv("SLIM_NO_MC") != nullptr;
    a.mc = 1;
    static const int mc_max = getenv("SLIM_MC_MAX") ? atoi(getenv("SLIM_MC_MAX")) : 1;   // multicast measured slower
    if (!no_mc && a.n_tiles > 1 && per_sm == 1) {
        for (int m = mc_max; m >= 2; --m)
            if (a.n_tiles % m == 0) {
                a.mc = m;
                break;
            }
    }
    if (a.mc > 1) {
        const int vt = a.m_tiles * (a.n_tiles / a.mc);
        int nclusters = ctx->num_sms / a.mc;
        if (nclusters > vt) nclusters = vt;
        grid = nclusters * a.mc;
    }
    double flops, bytes;
    conv_work(c, cc, ri, B, Ho, Wo, &flops, &bytes);
    if (ctx->trace) cudaMemsetAsync(ctx->trace, 0, 3584 * sizeof(unsigned long long), st);   // diagnostics (stem: 3584..)
    LaunchProf prof(ctx, st);
    cudaError_t e = launch_conv_umma(a, tA0, *tB0, tA1, *tB1, tRes, tOut, grid, st, ctx->pdl && !ctx->prof_on);
    prof.done(SLIM_K_CONV_UMMA, cc.seg, cc.layer, c.widths[cc.ri_in], c.widths[ri], B, flops, bytes);
    if (e != cudaSuccess)
        return fail(ctx, SLIM_ECUDA, "conv_umma launch (grid %d, cluster %d, smem %zu, n_tile %d, stages %d): %s", grid,
                    a.mc, smem, a.n_tile, a.n_stages, cudaGetErrorString(e));
    return SLIM_OK;
}

slim_status conv_f32(slim_ctx *ctx, cudaStream_t st, const ConvCall &cc, int ri, int B) {
    const slim_config &c = ctx->cfg;
    DevLayer &L = *cc.L;
    const int k = L.sh.k, s = L.sh.stride, pad = k / 2;
    ConvF32Args a{};
    a.x = static_cast<const float *>(cc.x);
    a.B = B;
    a.H = cc.H;
    a.W = cc.W;
    a.c_in = cc.c_in;
    a.w = static_cast<const float *>(L.w);
    a.cin_full = L.sh.cin;
    a.k = k;
    a.stride = s;
    a.pad = pad;
    a.Ho = (cc.H + 2 * pad - k) / s + 1;
    a.Wo = (cc.W + 2 * pad - k) / s + 1;
    a.c_out = slim_act_channels(c.widths[ri], L.sh.cout);
    a.scale0 = L.scale[ri];
    a.shift0 = L.shift[ri];
    if (cc.epi == EPI_BN_PROJ_RELU) {
        a.x1 = static_cast<const float *>(cc.xp);
        a.H1 = cc.Hp;
        a.W1 = cc.Wp;
        a.c_in1 = cc.c_in_p;
        a.stride1 = cc.Lp->sh.stride;
        a.w1 = static_cast<const float *>(cc.Lp->w);
        a.cin1_full = cc.Lp->sh.cin;
        a.scale1 = cc.Lp->scale[ri];
        a.shift1 = cc.Lp->shift[ri];
    }
    a.res = static_cast<const float *>(cc.res);
    a.out = static_cast<float *>(cc.out);
    a.epi = cc.epi;
    a.relu_lo = cc.relu_lo;
    a.ksplit = cc.f32_part ? f32_ksplit(c, cc.seg, c.widths[ri]) : 1;
    a.part = cc.f32_part;
    {   // SM share of this width (< 1, or SLIM_GRID_CAP): 2 resident GEMM CTAs per SM of the share,
        // persistent over tiles; at the full share: one CTA per tile (max_ctas = 0)
        const int cap = grid_cap(ctx, ri, ctx->num_sms, cc.seg);
        a.max_ctas = cap < ctx->num_sms ? 2 * cap : 0;
    }
    double flops, bytes;
    conv_work(c, cc, ri, B, a.Ho, a.Wo, &flops, &bytes);
    LaunchProf prof(ctx, st);
    cudaError_t e = launch_conv_f32(a, st);
    prof.done(SLIM_K_CONV_F32, cc.seg, cc.layer, c.widths[cc.ri_in], c.widths[ri], B, flops, bytes);
    if (e != cudaSuccess) return fail(ctx, SLIM_ECUDA, "conv_f32 launch: %s", cudaGetErrorString(e));
    return SLIM_OK;
}

slim_status check_sticky(slim_ctx *ctx) {
    if (ctx->sticky != SLIM_OK) return ctx->sticky;
    cudaError_t e = cudaPeekAtLastError();
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(ctx, SLIM_ECUDA, "asynchronous CUDA error: %s", cudaGetErrorString(e));
    }
    return SLIM_OK;
}

slim_status validate_fwd(slim_ctx *ctx, int seg, float r_prev, float r, int batch, const void *in, const void *out,
                         int *ri_prev, int *ri) {
    if (!ctx) return SLIM_EINVAL;
    const slim_config &c = ctx->cfg;
    if (seg < 0 || seg > 3) return fail(ctx, SLIM_EINVAL, "seg %d out of range", seg);
    if (batch < 1 || batch > c.max_batch) return fail(ctx, SLIM_EINVAL, "batch %d not in [1, %d]", batch, c.max_batch);
    *ri = width_index(c, r);
    if (*ri < 0) return fail(ctx, SLIM_EINVAL, "width %g not in the slimming set", r);
    *ri_prev = *ri;
    if (seg > 0) {
        *ri_prev = width_index(c, r_prev);
        if (*ri_prev < 0) return fail(ctx, SLIM_EINVAL, "r_prev %g not in the slimming set", r_prev);
    }
    if (!in || !out || !aligned16(in) || !aligned16(out)) return fail(ctx, SLIM_EINVAL, "in/out NULL or not 16-B aligned");
    if (!ctx->seg[seg].loaded) return fail(ctx, SLIM_ENOTLOADED, "segment %d not loaded", seg);
    return SLIM_OK;
}

// The segment schedule (O5/O6 in SURVEY §8(c)); all buffers validated by the caller.
// GroupNorm mode (reading R16): out = act(GN(y) [+ GN_p(yp)] [+ res]) over [B, H, H, C].
slim_status gn_apply(slim_ctx *ctx, cudaStream_t st, int seg, int layer, const DevLayer &L, const DevLayer *Lp,
                     int ri, int B, int H, int C, const void *y, const void *yp, const void *res, void *out, bool relu,
                     float *pool_out = nullptr) {
    const slim_config &c = ctx->cfg;
    GnArgs g{};
    g.y = y;
    g.yp = yp;
    g.res = res;
    g.gamma = L.gn_gamma[ri];
    g.beta = L.gn_beta[ri];
    if (yp) {
        g.gamma_p = Lp->gn_gamma[ri];
        g.beta_p = Lp->gn_beta[ri];
    }
    g.out = out;
    g.B = B;
    g.HW = H * H;
    g.C = C;
    g.cpg = c.gn_group_channels;
    g.gpc = gn_groups_per_cta(B, g.HW, C, g.cpg, c.dtype == SLIM_FP32);
    g.eps = c.bn_eps;
    g.relu_lo = relu ? 0.f : -INFINITY;
    g.pool_out = pool_out;   // the network's last GN: average pool fp32 [B][C] instead of the activation
    {   // SM share of this width: gn_mult CTAs per SM of the share (persistent over items); 0 = uncapped
        static const int gn_mult = getenv("SLIM_GN_CAP_MULT") ? atoi(getenv("SLIM_GN_CAP_MULT")) : 0;   // measured: uncapped 716k, x3 699k, x6 717k
        const int cap = grid_cap(ctx, ri, 1 << 30, seg);
        g.max_ctas = (gn_mult > 0 && cap < (1 << 30)) ? gn_mult * cap : 0;
    }
    const double eb = static_cast<double>(elem_bytes(c));
    const double n = static_cast<double>(B) * H * H * C;
    const double flops = 8.0 * n * (yp ? 2 : 1);   // 2 statistics passes + apply, per input tensor
    const double bytes = eb * n * (2 + (yp ? 1 : 0) + (res ? 1 : 0)) + 8.0 * C * (yp ? 2 : 1);
    LaunchProf prof(ctx, st);
    const cudaError_t e = launch_gn(g, c.dtype == SLIM_FP32, st, ctx->pdl && !ctx->prof_on);
    prof.done(SLIM_K_GN, seg, layer, c.widths[ri], c.widths[ri], B, flops, bytes);
    if (e != cudaSuccess) return fail(ctx, SLIM_ECUDA, "gn launch: %s", cudaGetErrorString(e));
    return SLIM_OK;
}

// GroupNorm mode, fast path: the conv wrote statistics partials (ConvCall::gn_stats); apply elementwise.
slim_status gn_apply_part(slim_ctx *ctx, cudaStream_t st, int seg, int layer, const DevLayer &L, int ri, int B, int H,
                          int C, const void *y, const float2 *part, int tiles_per_img, const void *res, void *out,
                          float *pool_out = nullptr) {
    const slim_config &c = ctx->cfg;
    GnPartArgs g{};
    g.y = static_cast<const uint16_t *>(y);
    g.part = part;
    g.res = static_cast<const uint16_t *>(res);
    g.gamma = L.gn_gamma[ri];
    g.beta = L.gn_beta[ri];
    g.out = static_cast<uint16_t *>(out);
    g.pool_out = pool_out;
    g.B = B;
    g.HW = H * H;
    g.C = C;
    g.tiles_per_img = tiles_per_img;
    g.part_count = static_cast<float>(g.HW / tiles_per_img * 16);
    g.eps = c.bn_eps;
    g.relu_lo = 0.f;
    {
        const int cap = grid_cap(ctx, ri, ctx->num_sms, seg);
        g.max_ctas = cap < ctx->num_sms ? 8 * cap : 0;
    }
    const double n = static_cast<double>(B) * H * H * C;
    const double flops = 4.0 * n;
    const double bytes = 2.0 * n * (2 + (res ? 1 : 0)) + 8.0 * C;
    LaunchProf prof(ctx, st);
    const cudaError_t e = launch_gn_apply_part(g, st, ctx->pdl && !ctx->prof_on);
    prof.done(SLIM_K_GN, seg, layer, c.widths[ri], c.widths[ri], B, flops, bytes);
    if (e != cudaSuccess) return fail(ctx, SLIM_ECUDA, "gn apply launch: %s", cudaGetErrorString(e));
    return SLIM_OK;
}

slim_status run_segment(slim_ctx *ctx, int seg, int ri_prev, int ri, int B, const void *in, void *out, void *ws,
                        cudaStream_t st) {
    const slim_config &c = ctx->cfg;
    DevSegment &S = ctx->seg[seg];
    const bool bf = c.dtype == SLIM_BF16;
    const double eb = static_cast<double>(elem_bytes(c));
    const float r = c.widths[ri];
    const int H = seg_hw(c, seg);
    const bool gn = c.norm == SLIM_NORM_GN;
    const float relu_lo = gn ? -INFINITY : 0.f;   // GN: convs store the raw pre-norm output
    float *gn_pooled = nullptr;                    // GN: the last GN's fused average pool (fp32 [B][C])
    const int C = slim_act_channels(r, c.base_channels[seg]);
    const size_t buf = round256(act_bytes(c, seg, r, B));
    char *bufs[3] = {static_cast<char *>(ws), static_cast<char *>(ws) + buf, static_cast<char *>(ws) + 2 * buf};
    // FP32 mode: split-K partials after the buffers (f32_part_bytes)
    float *f32_part = (!bf && f32_ksplit(c, seg, r) > 1)
                          ? reinterpret_cast<float *>(static_cast<char *>(ws) + 3 * buf + gn_part_bytes(c, seg, r, B) +
                                                      tile_flag_bytes(c, B))
                          : nullptr;
    const void *cur = in;
    int curH = (seg == 0) ? H : (H * 2);
    int curC = (seg == 0) ? c.in_channels : slim_act_channels(c.widths[ri_prev], c.base_channels[seg - 1]);
    // segment 0 at a narrow width: stem + both blocks in one kernel, activations in shared memory
    // (kernels_fused.cu; bit-identical to the per-layer kernels below).  SLIM_NO_FUSED=1: per-layer path.
    static const bool no_fused = getenv("SLIM_NO_FUSED") != nullptr;
    // GroupNorm: fused too (two-pass statistics in the kernel), but only while the width has the GPU to
    // itself -- under SM partitioning the two-pass kernel holds its SMs long enough to slow the concurrent
    // step (GN CFG2 668 k vs 707 k images/s, tools/gpu_runs/r02_gnfused.sh)
    static const bool no_fused_gn = getenv("SLIM_NO_FUSED_GN") != nullptr;
    const bool seg0_partitioned = grid_cap(ctx, ri, ctx->num_sms, 0) < ctx->num_sms;
    if (seg == 0 && bf && (!gn || (!no_fused_gn && c.gn_group_channels == 16 && !seg0_partitioned)) && !no_fused &&
        (C == 16 || C == 32) &&
        C == slim_channels(r, c.base_channels[0]) && H == 32 && c.in_channels == 3 && c.blocks_per_seg[0] == 2 &&
        S.L[1].sh.cin % 8 == 0) {
        FusedSeg0Args fa{};
        fa.in = static_cast<const uint16_t *>(in);
        fa.out = static_cast<uint16_t *>(out);
        fa.B = B;
        fa.c0 = C;
        fa.cin_full = S.L[1].sh.cin;
        for (int l = 0; l < 4; ++l) fa.w[l] = static_cast<const uint16_t *>(S.L[1 + l].w);
        fa.stem_b = S.L[0].stem_b;
        fa.trace = ctx->trace ? ctx->trace + 8192 : nullptr;
        fa.gn = gn ? 1 : 0;   // GroupNorm: the kernel's two-pass statistics; scale/shift carry gamma/beta
        fa.eps = c.bn_eps;
        for (int l = 0; l < 5; ++l) {
            fa.scale[l] = gn ? S.L[l].gn_gamma[ri] : S.L[l].scale[ri];
            fa.shift[l] = gn ? S.L[l].gn_beta[ri] : S.L[l].shift[ri];
        }
        const double pix = static_cast<double>(B) * H * H;
        const double flops = 2.0 * pix * C * 9 * (c.in_channels + 4.0 * C);
        // the SURVEY §8(d) roofline's layer-materialised bytes (each layer reads its input, residual and
        // weights and writes its output), so the fused kernel is measured against the same roofline as
        // the per-layer kernels; its compulsory traffic is only in + out + weights
        const double bytes = eb * pix * (c.in_channels + C) + eb * 27.0 * C +                  // stem
                             4.0 * (eb * pix * 2.0 * C + eb * 9.0 * C * C) + 2.0 * eb * pix * C +   // 4 convs, 2 residuals
                             48.0 * C;
        // small batches: a cluster of 8 CTAs per image (one 4-row tile each, halo rows through DSMEM) --
        // a layer is then one tile's MMA + epilogue instead of eight; one CTA per image once 8 B CTAs no
        // longer fit the SMs (or the width shares the GPU).  Batch-independent either way (same
        // arithmetic).  SLIM_SEG0_CLUSTER=0/8 forces.
        static const int cl_env = getenv("SLIM_SEG0_CLUSTER") ? atoi(getenv("SLIM_SEG0_CLUSTER")) : -1;
        const int cap_sms = grid_cap(ctx, ri, ctx->num_sms, 0);
        fa.cluster = cl_env >= 0 ? (cl_env == 8 ? 8 : 1) : (8 * B <= cap_sms && cap_sms == ctx->num_sms ? 8 : 1);
        int grid = std::min(B, ctx->num_sms / fa.cluster);
        if (fa.cluster == 1) grid = grid_cap(ctx, ri, grid, 0);
        LaunchProf prof(ctx, st);
        const cudaError_t e = launch_seg0_fused(fa, grid, st, ctx->pdl && !ctx->prof_on);
        prof.done(SLIM_K_SEG_FUSED, 0, 0, r, r, B, flops, bytes);
        if (e != cudaSuccess) return fail(ctx, SLIM_ECUDA, "fused segment-0 launch: %s", cudaGetErrorString(e));
        return SLIM_OK;
    }
    // segments 1-3 at a narrow width: both blocks in one kernel (kernels_fused.cu) wherever the (r_prev, r)
    // working set fits in shared memory (the weight image then exists): measured faster than the per-layer
    // kernels at B = 8 and 128 for every such case (profiles/r02_fused_micro.txt).  SLIM_FUSED_SEGS (bit s =
    // segment s) restricts it (A/B).
    static const int fused_env = getenv("SLIM_FUSED_SEGS") ? atoi(getenv("SLIM_FUSED_SEGS")) : 0xE;
    // While the width's instance shares the GPU with concurrent instances (SM share < 1, the CFG2 step),
    // segments 1-3 take the per-layer kernels: a fused unit is a long per-CTA latency chain that holds its
    // SMs (large smem) for most of the step and starves the wide instances' kernels -- measured 1.07 M
    // (fused, capped to the share) / 1.12 M (fused, uncapped) vs 1.27 M images/s (per-layer) for the
    // 4-width step (tools/gpu_runs/r02_ab_fused2.sh).  SLIM_FUSED_PART (A/B): 0 = that (default),
    // 1 = fused and capped to the share, 2 = fused and uncapped.
    static const int fused_part = getenv("SLIM_FUSED_PART") ? atoi(getenv("SLIM_FUSED_PART")) : 0;
    const bool partitioned = grid_cap(ctx, ri, ctx->num_sms, seg) < ctx->num_sms;
    // Large batches (BN mode): a fused unit is a per-CTA latency chain, so once the units fill the SMs
    // several times over the per-layer kernels' throughput wins (profiles/r02_fused_thresh.txt, each
    // width alone): seg 1 C <= 32 fused up to B = 1024, C = 64 up to 192; seg 2 C <= 64 up to 512,
    // C = 128 up to 128; seg 3 up to 256.  Both paths are bit-identical, so this is a pure speed choice.
    // SLIM_FUSED_BMAX (A/B) overrides the limit for every segment (0 = no limit).
    static const int bmax_env = getenv("SLIM_FUSED_BMAX") ? atoi(getenv("SLIM_FUSED_BMAX")) : -1;
    const int fused_bmax = bmax_env >= 0 ? (bmax_env ? bmax_env : (1 << 30))
                           : gn ? (1 << 30)
                           : seg == 1 ? (C <= 32 ? 1024 : 192)
                           : seg == 2 ? (C <= 64 ? 512 : 128)
                                      : 256;
    const bool fused_on = ((fused_env >> seg) & 1) != 0 && !(partitioned && fused_part == 0) && B <= fused_bmax;
    // GroupNorm: the kernel's two-pass statistics (per image and 16-channel group), same condition
    if (seg > 0 && bf && (!gn || !no_fused_gn) && !no_fused && fused_on && S.fimg[ri_prev][ri]) {
        FusedSegArgs fa{};
        fa.in = static_cast<const uint16_t *>(in);
        fa.B = B;
        fa.CI = curC;
        fa.wimg = static_cast<const uint8_t *>(S.fimg[ri_prev][ri]);
        fa.trace = ctx->trace ? ctx->trace + 8192 + 64 : nullptr;
        const bool last = seg == 3;
        float *pooled = nullptr;
        if (last) pooled = reinterpret_cast<float *>(bufs[0]);   // fp32 [B][C] for the FC
        else fa.out = static_cast<uint16_t *>(out);
        fa.pool_out = pooled;
        fa.gn = gn ? 1 : 0;
        fa.eps = c.bn_eps;
        for (int l = 0; l < 5; ++l) {
            fa.scale[l] = gn ? S.L[l].gn_gamma[ri] : S.L[l].scale[ri];
            fa.shift[l] = gn ? S.L[l].gn_beta[ri] : S.L[l].shift[ri];
        }
        const int G = seg == 1 ? 1 : (seg == 2 ? 2 : 8);
        const double pix = static_cast<double>(B) * H * H;
        const double flops = 2.0 * pix * C * (9.0 * curC + 27.0 * C + curC);
        // layer-materialised bytes (SURVEY §8(d) roofline, as the per-layer kernels count them)
        const double in_b = eb * B * 4.0 * H * H * curC, act = eb * pix * C;
        const double bytes = (in_b + act + eb * 9.0 * curC * C) +                  // b0c1 (stride 2)
                             (act + in_b + act + eb * (9.0 * C * C + curC * C)) +   // b0c2 + projection
                             (2.0 * act + eb * 9.0 * C * C) +                       // b1c1
                             (3.0 * act + eb * 9.0 * C * C) + 40.0 * C;            // b1c2 + residual
        const int P = segn_fused_cluster(seg, C);
        int grid = std::min((B + G - 1) / G, ctx->num_sms / P);   // clusters (units in flight)
        if (fused_part != 2) grid = std::max(1, grid_cap(ctx, ri, grid * P, seg) / P);
        LaunchProf prof(ctx, st);
        const cudaError_t e = launch_segn_fused(fa, seg, C, grid, st, ctx->pdl && !ctx->prof_on);
        prof.done(SLIM_K_SEG_FUSED, seg, 0, c.widths[ri_prev], r, B, flops, bytes);
        if (e != cudaSuccess) return fail(ctx, SLIM_ECUDA, "fused segment-%d launch: %s", seg, cudaGetErrorString(e));
        if (last) {   // the head: FC on the pooled features
            const double K = c.num_classes;
            LaunchProf prof2(ctx, st);
            const cudaError_t e2 = launch_fc_f32(pooled, S.fc_w, S.fc_b, static_cast<float *>(out), B, C,
                                                 c.base_channels[3], c.num_classes, st, ctx->pdl && !ctx->prof_on);
            prof2.done(SLIM_K_HEAD, 3, -1, r, r, B, 2.0 * B * C * K, 4.0 * B * C + 4.0 * K * (C + 1) + 4.0 * B * K);
            if (e2 != cudaSuccess) return fail(ctx, SLIM_ECUDA, "head launch: %s", cudaGetErrorString(e2));
        }
        return SLIM_OK;
    }
    if (seg == 0) {
        DevLayer &Ls = S.L[0];
        const double pix = static_cast<double>(B) * H * H;
        const double flops = 2.0 * pix * C * 9 * c.in_channels;
        const double bytes = eb * pix * (c.in_channels + C) + 4.0 * C * 9 * c.in_channels + 8.0 * C;
        cudaError_t e;
        if (bf) {
            StemArgs sa{};
            sa.in = static_cast<const uint16_t *>(in);
            sa.w = static_cast<const float *>(Ls.w);
            sa.b_img = Ls.stem_b;
            sa.w_stride = 9 * Ls.sh.cin;
            sa.scale = Ls.scale[ri];
            sa.shift = Ls.shift[ri];
            sa.B = B;
            sa.H = H;
            sa.W = H;
            sa.cimg = c.in_channels;
            sa.c0 = C;
            sa.tile_rows = kTileM / H;
            sa.m_tiles = B * (H / sa.tile_rows);
            sa.tmem_cols = C <= 16 ? 64 : 128;   // two accumulator stages of round32(C) columns
            sa.trace = ctx->trace;
            sa.relu_lo = relu_lo;
            if (ctx->trace) cudaMemsetAsync(ctx->trace + 3584, 0, 512 * sizeof(unsigned long long), st);
            CUtensorMap tIn, tOut;
            {   // the image as flat rows: (W*cimg, H, B), box = the tile's rows plus the 3x3 halo
                const cuuint64_t rowe = static_cast<cuuint64_t>(H) * c.in_channels;
                cuuint64_t dims[3] = {rowe, (cuuint64_t)H, (cuuint64_t)B};
                cuuint64_t strides[2] = {rowe * 2, rowe * 2 * H};
                cuuint32_t box[3] = {(cuuint32_t)rowe, (cuuint32_t)(sa.tile_rows + 2), 1};
                cuuint32_t est[3] = {1, 1, 1};
                if (!encode_map(ctx, &tIn, in, 3, dims, strides, box, est, false))
                    return fail(ctx, SLIM_ECUDA, "cuTensorMapEncodeTiled(stem in) failed");
            }
            if (!encode_act(ctx, &tOut, bufs[0], B, H, H, C, H, sa.tile_rows, 1, 1))
                return fail(ctx, SLIM_ECUDA, "cuTensorMapEncodeTiled(stem out) failed");
            // persistent: one CTA per SM, halo fetch / im2col / MMA / store of consecutive tiles overlap
            int grid = ctx->num_sms;
            if (grid > sa.m_tiles) grid = sa.m_tiles;
            grid = grid_cap(ctx, ri, grid, 0);
            LaunchProf prof(ctx, st);
            e = launch_stem_umma(sa, tIn, tOut, grid, st, ctx->pdl && !ctx->prof_on);
            prof.done(SLIM_K_STEM, 0, 0, r, r, B, flops, bytes);
        } else {
            LaunchProf prof(ctx, st);
            e = launch_stem_f32(static_cast<const float *>(in), static_cast<const float *>(Ls.w), Ls.sh.cin,
                                Ls.scale[ri], Ls.shift[ri], reinterpret_cast<float *>(bufs[0]), B, H, H,
                                c.in_channels, C, st, relu_lo);
            prof.done(SLIM_K_STEM, 0, 0, r, r, B, flops, bytes);
        }
        if (e != cudaSuccess) return fail(ctx, SLIM_ECUDA, "stem launch: %s", cudaGetErrorString(e));
        if (gn) {   // h = ReLU(GN(stem(x))), in place
            const slim_status gs = gn_apply(ctx, st, 0, 0, Ls, nullptr, ri, B, H, C, bufs[0], nullptr, nullptr, bufs[0], true);
            if (gs) return gs;
        }
        cur = bufs[0];
        curH = H;
        curC = C;
    }
    const int nb = c.blocks_per_seg[seg];
    // Tile-granular dependencies inside a segment (BN, bf16, two blocks, all four convs on the halo kernel
    // with one M tiling): block 1's convs start a tile as soon as the tiles of the previous conv it reads
    // are finished, instead of waiting for that whole grid; block 0's conv1 clears the counters.
    // Opt-in (SLIM_TILE_FLAGS=1): bitwise equal, but measured slower (r = 1 B = 128 segment 0 61 -> 70 us,
    // B = 1024 357 -> 407 us, CFG2 1.21 -> 1.11 M images/s) with serial acquires, parallel relaxed polls +
    // one acquire fence, and the producer's publication two tiles behind alike: the cost grows with the
    // tile count (~0.45 us per tile of a flagged layer), i.e. it is per tile, not per boundary; removing
    // either async-proxy fence (an A/B only -- they are needed for correctness) changes nothing, so the
    // cost is structural (the dependents' producers start loading while the previous grid still runs);
    // and the persistent one-CTA-per-SM grids only overlap at their tails anyway.
    static const bool tile_flags = getenv("SLIM_TILE_FLAGS") && atoi(getenv("SLIM_TILE_FLAGS")) != 0;
    uint32_t *flags = nullptr;
    int flag_nt[4] = {0, 0, 0, 0}, flag_m = 0;
    if (tile_flags && bf && !gn && nb == 2 && !ctx->prof_on) {
        bool ok = true;
        const void *X = cur;
        int xH = curH, xC = curC;
        for (int b = 0; b < 2 && ok; ++b) {
            const BlockIdx bi = block_layers(c, seg, b);
            const bool down = seg > 0 && b == 0;
            ConvCall d1;   // shapes only (the pointers are placeholders: nothing is launched)
            d1.seg = seg;
            d1.layer = bi.c1;
            d1.L = &S.L[bi.c1];
            d1.ri_in = down ? ri_prev : ri;
            d1.x = X;
            d1.H = d1.W = xH;
            d1.c_in = xC;
            d1.out = bufs[0];
            d1.epi = EPI_BN_RELU;
            ConvCall d2 = d1;
            d2.layer = bi.c2;
            d2.L = &S.L[bi.c2];
            d2.ri_in = ri;
            d2.x = bufs[0];
            d2.H = d2.W = H;
            d2.c_in = C;
            if (seg == 3 && b == 1 && H * H <= 32 && 32 % (H * H) == 0) d2.pool_out = reinterpret_cast<float *>(bufs[1]);
            if (down) {
                d2.epi = EPI_BN_PROJ_RELU;
                d2.Lp = &S.L[bi.sc];
                d2.layer_p = bi.sc;
                d2.ri_in_p = ri_prev;
                d2.xp = X;
                d2.Hp = d2.Wp = xH;
                d2.c_in_p = xC;
            } else {
                d2.epi = EPI_BN_ADD_RELU;
                d2.res = X;
            }
            HaloArgs h1{}, h2{};
            d1.dry = &h1;
            d2.dry = &h2;
            ok = conv_halo_bf16(ctx, st, d1, ri, B) == SLIM_OK && conv_halo_bf16(ctx, st, d2, ri, B) == SLIM_OK;
            if (ok) {
                flag_nt[2 * b] = h1.n_tiles;
                flag_nt[2 * b + 1] = h2.n_tiles;
                if (h1.m_tiles != h2.m_tiles || (b == 1 && h1.m_tiles != flag_m)) ok = false;
                flag_m = h1.m_tiles;
            }
            X = bufs[1];
            xH = H;
            xC = C;
        }
        if (ok && 2 * static_cast<size_t>(flag_m) * sizeof(uint32_t) <= tile_flag_bytes(c, B))
            flags = reinterpret_cast<uint32_t *>(static_cast<char *>(ws) + 3 * buf + gn_part_bytes(c, seg, r, B));
    }
    for (int b = 0; b < nb; ++b) {
        const BlockIdx bi = block_layers(c, seg, b);
        const bool down = seg > 0 && b == 0;
        const int ri_in = down ? ri_prev : ri;
        // pick T and dst among the 3 workspace buffers, never aliasing cur
        char *free_[3];
        int nf = 0;
        for (int i = 0; i < 3; ++i)
            if (bufs[i] != cur) free_[nf++] = bufs[i];
        char *T = free_[0];
        void *dst = (b == nb - 1 && seg < 3) ? out : free_[1];
        ConvCall c1;   // t = relu(BN1(conv3x3_s(x)))
        c1.seg = seg;
        c1.layer = bi.c1;
        c1.L = &S.L[bi.c1];
        c1.ri_in = ri_in;
        c1.x = cur;
        c1.H = c1.W = curH;
        c1.c_in = curC;
        c1.out = T;
        c1.epi = EPI_BN_RELU;
        c1.f32_part = f32_part;
        // the network's last conv pools in its epilogue (BF16 mode): the segment-3 output
        // never goes to memory; the head is then the FC alone
        const bool fuse_pool = !gn && bf && seg == 3 && b == nb - 1 && H * H <= 32 && 32 % (H * H) == 0;
        ConvCall c2;   // out = relu(BN2(conv3x3(t)) + shortcut)
        c2.seg = seg;
        c2.layer = bi.c2;
        c2.L = &S.L[bi.c2];
        c2.ri_in = ri;
        c2.x = T;
        c2.H = c2.W = H;
        c2.c_in = C;
        c2.out = dst;
        c2.f32_part = f32_part;
        if (fuse_pool) c2.pool_out = reinterpret_cast<float *>(dst);
        if (down) {
            c2.epi = EPI_BN_PROJ_RELU;
            c2.Lp = &S.L[bi.sc];
            c2.layer_p = bi.sc;
            c2.ri_in_p = ri_in;
            c2.xp = cur;
            c2.Hp = c2.Wp = curH;
            c2.c_in_p = curC;
        } else {
            c2.epi = EPI_BN_ADD_RELU;
            c2.res = cur;
        }
        // GroupNorm in the conv epilogue where a tile holds whole images (segments 2-3, halo kernel):
        // t = ReLU(GN1(conv1(x))) and out = ReLU(GN2(conv2(t)) + [GN_p(proj(x)) | x]) [pooled] -- two
        // launches per block instead of four or five.  SLIM_GN_EPI=0 keeps the separate GN kernels (A/B).
        static const bool gn_epi = !getenv("SLIM_GN_EPI") || atoi(getenv("SLIM_GN_EPI")) != 0;
        bool gn_c1_done = false;
        // Segment 1 (two M tiles per image) as image pairs -- one CTA takes both tiles, both accumulators
        // resident -- is opt-in (SLIM_GN_PAIRS=1): parity green but measured slower (r = 1 GN seg 1
        // 98 -> 103 us, GN CFG2 766 k -> 650 k: the pair serialises MMA and epilogue per image)
        static const bool gn_pairs = getenv("SLIM_GN_PAIRS") && atoi(getenv("SLIM_GN_PAIRS")) != 0;
        if (gn && bf && gn_epi && (H * H < kTileM || (gn_pairs && H * H == 2 * kTileM))) {
            ConvCall g1 = c1;
            g1.gn_fuse = true;
            const slim_status sg = conv_halo_bf16(ctx, st, g1, ri, B);
            if (sg != SLIM_OK && sg != SLIM_EUNSUPPORTED) return sg;
            gn_c1_done = sg == SLIM_OK;
            if (gn_c1_done) {
                ConvCall g2 = c2;
                g2.gn_fuse = true;
                const bool last = seg == 3 && b == nb - 1;
                if (last) g2.pool_out = reinterpret_cast<float *>(dst);   // the head is then the FC alone
                const slim_status s2 = conv_halo_bf16(ctx, st, g2, ri, B);
                if (s2 != SLIM_OK && s2 != SLIM_EUNSUPPORTED) return s2;
                if (s2 == SLIM_OK) {
                    if (last) gn_pooled = reinterpret_cast<float *>(dst);
                    cur = dst;
                    curH = H;
                    curC = C;
                    continue;
                }
            }
        }
        if (gn) {
            // t = ReLU(GN1(conv1(x))): conv writes raw into T, GN in place.  u = conv2(t) raw into dst;
            // the projection (raw) reuses T once conv2 has read it; then dst = ReLU(GN2(u) + shortcut).
            // Where the conv is the halo kernel it also writes the GroupNorm statistics partials (part),
            // and the GN is an elementwise pass over them (gn_apply_part) instead of a reduction kernel.
            float2 *part = bf ? reinterpret_cast<float2 *>(static_cast<char *>(ws) + 3 * buf) : nullptr;
            c1.relu_lo = relu_lo;
            c1.gn_part = part;
            slim_status s1 = SLIM_OK;
            if (!gn_c1_done) {   // (else conv1 already wrote T = ReLU(GN1(.)) above)
                s1 = bf ? conv_bf16(ctx, st, c1, ri, B) : conv_f32(ctx, st, c1, ri, B);
                if (s1) return s1;
                s1 = c1.gn_stats ? gn_apply_part(ctx, st, seg, bi.c1, S.L[bi.c1], ri, B, H, C, T, part, c1.gn_tiles_per_img,
                                                 nullptr, T)
                                 : gn_apply(ctx, st, seg, bi.c1, S.L[bi.c1], nullptr, ri, B, H, C, T, nullptr, nullptr, T, true);
                if (s1) return s1;
            }
            ConvCall u = c2;
            u.epi = EPI_BN_RELU;
            u.relu_lo = relu_lo;
            u.res = nullptr;
            u.Lp = nullptr;
            u.pool_out = nullptr;
            u.gn_part = down ? nullptr : part;   // (a down block's GN pairs u with the projection's GN)
            s1 = bf ? conv_bf16(ctx, st, u, ri, B) : conv_f32(ctx, st, u, ri, B);
            if (s1) return s1;
            const void *yp = nullptr;
            if (down) {
                ConvCall p;   // 1x1 stride-2 projection, raw
                p.seg = seg;
                p.layer = bi.sc;
                p.L = &S.L[bi.sc];
                p.ri_in = ri_in;
                p.x = cur;
                p.H = p.W = curH;
                p.c_in = curC;
                p.out = T;
                p.epi = EPI_BN_RELU;
                p.relu_lo = relu_lo;
                p.f32_part = f32_part;
                s1 = bf ? conv_bf16(ctx, st, p, ri, B) : conv_f32(ctx, st, p, ri, B);
                if (s1) return s1;
                yp = T;
            }
            // the network's last GN pools in place of its store (the head is then the FC alone); the
            // pooled fp32 [B][C] goes to a buffer this GN does not read: T (free unless it holds the
            // projection), else the block input if it is a workspace buffer (never the caller's `in`)
            if (seg == 3 && b == nb - 1) {
                void *pb = !down ? static_cast<void *>(T) : (cur != in ? const_cast<void *>(cur) : nullptr);
                gn_pooled = static_cast<float *>(pb);
            }
            s1 = u.gn_stats ? gn_apply_part(ctx, st, seg, bi.c2, S.L[bi.c2], ri, B, H, C, dst, part, u.gn_tiles_per_img,
                                            cur, dst, gn_pooled)
                            : gn_apply(ctx, st, seg, bi.c2, S.L[bi.c2], down ? &S.L[bi.sc] : nullptr, ri, B, H, C, dst, yp,
                                       down ? nullptr : cur, dst, true, gn_pooled);
            if (s1) return s1;
            cur = dst;
            curH = H;
            curC = C;
            continue;
        }
        if (flags) {   // layers: b0.c1 clears, b0.c2 -> F0 -> b1.c1 -> F1 -> b1.c2
            uint32_t *F0 = flags, *F1 = flags + flag_m;
            if (b == 0) {
                c1.flag_zero = flags;
                c1.flag_zero_n = 2 * flag_m;
                c2.flag_out = F0;
            } else {
                c1.flag_in = F0;
                c1.flag_in_target = flag_nt[1];
                c1.flag_out = F1;
                c2.flag_in = F1;
                c2.flag_in_target = flag_nt[2];
            }
            slim_status s1 = conv_halo_bf16(ctx, st, c1, ri, B);
            if (s1) return s1 == SLIM_EUNSUPPORTED ? fail(ctx, SLIM_ECUDA, "tile flags: halo declined a planned layer") : s1;
            slim_status s2 = conv_halo_bf16(ctx, st, c2, ri, B);
            if (s2) return s2 == SLIM_EUNSUPPORTED ? fail(ctx, SLIM_ECUDA, "tile flags: halo declined a planned layer") : s2;
            cur = dst;
            curH = H;
            curC = C;
            continue;
        }
        slim_status s1 = bf ? conv_bf16(ctx, st, c1, ri, B) : conv_f32(ctx, st, c1, ri, B);
        if (s1) return s1;
        slim_status s2 = bf ? conv_bf16(ctx, st, c2, ri, B) : conv_f32(ctx, st, c2, ri, B);
        if (s2) return s2;
        cur = dst;
        curH = H;
        curC = C;
    }
    if (seg == 3) {
        const double K = c.num_classes;
        const bool pooled = gn ? gn_pooled != nullptr : (bf && H * H <= 32 && 32 % (H * H) == 0);   // fuse_pool
        if (gn_pooled) cur = gn_pooled;
        const double flops = 2.0 * B * C * K + (pooled ? 0.0 : static_cast<double>(B) * H * H * C);
        const double bytes = (pooled ? 4.0 * B * C : eb * B * H * H * C) + 4.0 * K * (C + 1) + 4.0 * B * K;
        LaunchProf prof(ctx, st);
        const bool pdl = ctx->pdl && !ctx->prof_on;
        cudaError_t e = pooled ? launch_fc_f32(static_cast<const float *>(cur), S.fc_w, S.fc_b, static_cast<float *>(out),
                                               B, C, c.base_channels[3], c.num_classes, st, pdl)
                        : bf ? launch_head_bf16(static_cast<const uint16_t *>(cur), S.fc_w, S.fc_b,
                                                static_cast<float *>(out), B, H * H, C, c.base_channels[3],
                                                c.num_classes, st, pdl)
                             : launch_head_f32(static_cast<const float *>(cur), S.fc_w, S.fc_b,
                                               static_cast<float *>(out), B, H * H, C, c.base_channels[3],
                                               c.num_classes, st, pdl);
        prof.done(SLIM_K_HEAD, 3, -1, r, r, B, flops, bytes);
        if (e != cudaSuccess) return fail(ctx, SLIM_ECUDA, "head launch: %s", cudaGetErrorString(e));
    }
    return SLIM_OK;
}

// Graph mode: replay a captured launch sequence for an identical argument list.
template <class F>
slim_status run_graphed(slim_ctx *ctx, const std::string &key, cudaStream_t st, F &&body) {
    if (!ctx->graph_mode || ctx->prof_on) return body(st);
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return body(st);
    std::lock_guard<std::mutex> g(ctx->graph_mu);
    auto it = ctx->graphs.find(key);
    if (it == ctx->graphs.end()) {
        const uint64_t l0 = ctx->launches.load();
        CUDA_TRY(ctx, cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal));
        slim_status s = body(ctx->cap_stream);
        cudaGraph_t graph = nullptr;
        cudaError_t e = cudaStreamEndCapture(ctx->cap_stream, &graph);
        if (s != SLIM_OK) {
            if (graph) cudaGraphDestroy(graph);
            return s;
        }
        if (e != cudaSuccess) return fail(ctx, SLIM_ECUDA, "graph capture: %s", cudaGetErrorString(e));
        cudaGraphExec_t exec = nullptr;
        e = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) return fail(ctx, SLIM_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
        const uint64_t n = ctx->launches.load() - l0;
        ctx->launches -= n;   // counted when replayed
        it = ctx->graphs.emplace(key, slim_ctx::GraphEntry{exec, n}).first;
    }
    CUDA_TRY(ctx, cudaGraphLaunch(it->second.exec, st));
    ctx->launches += it->second.n_kernels;
    return SLIM_OK;
}

template <class... T>
std::string make_key(T... v) {
    std::string k;
    int dummy[] = {(k.append(reinterpret_cast<const char *>(&v), sizeof(v)), 0)...};
    (void)dummy;
    return k;
}

void free_segment(DevSegment &S) {
    for (int l = 0; l < S.n_conv; ++l) {
        DevLayer &L = S.L[l];
        cudaFree(L.w);
        cudaFree(L.stem_b);
        for (int i = 0; i < kMaxW; ++i) {
            cudaFree(L.scale[i]);
            cudaFree(L.shift[i]);
            cudaFree(L.gn_gamma[i]);
            cudaFree(L.gn_beta[i]);
        }
        L = DevLayer{};
    }
    cudaFree(S.fc_w);
    cudaFree(S.fc_b);
    for (int i = 0; i < kMaxW; ++i)
        for (int j = 0; j < kMaxW; ++j) cudaFree(S.fimg[i][j]);
    S = DevSegment{};
}

}  // namespace

// =============================================================================
extern "C" {

int slim_version(void) { return 1; }

const char *slim_status_str(slim_status s) {
    switch (s) {
        case SLIM_OK: return "SLIM_OK";
        case SLIM_EINVAL: return "SLIM_EINVAL";
        case SLIM_ENOTLOADED: return "SLIM_ENOTLOADED";
        case SLIM_ENOMEM: return "SLIM_ENOMEM";
        case SLIM_ECUDA: return "SLIM_ECUDA";
        case SLIM_EUNSUPPORTED: return "SLIM_EUNSUPPORTED";
    }
    return "unknown";
}

void slim_default_config(slim_config *cfg) {
    std::memset(cfg, 0, sizeof *cfg);
    cfg->n_widths = 4;
    cfg->widths[0] = 0.25f;
    cfg->widths[1] = 0.5f;
    cfg->widths[2] = 0.75f;
    cfg->widths[3] = 1.0f;
    for (int s = 0; s < 4; ++s) cfg->blocks_per_seg[s] = 2;
    cfg->base_channels[0] = 64;
    cfg->base_channels[1] = 128;
    cfg->base_channels[2] = 256;
    cfg->base_channels[3] = 512;
    cfg->in_channels = 3;
    cfg->num_classes = 100;
    cfg->image_hw = 32;
    cfg->max_batch = 4096;
    cfg->bn_eps = 1e-5f;
    cfg->dtype = SLIM_BF16;
    cfg->norm = SLIM_NORM_BN;
    cfg->gn_group_channels = 16;
}

slim_status slim_create(int device, const slim_config *cfg, slim_ctx **out) {
    if (!out) return SLIM_EINVAL;
    *out = nullptr;
    if (!cfg) return SLIM_EINVAL;
    const slim_config &c = *cfg;
    if (c.n_widths < 1 || c.n_widths > kMaxW) return SLIM_EINVAL;
    for (int i = 0; i < c.n_widths; ++i) {
        if (!(c.widths[i] > 0.f && c.widths[i] <= 1.f)) return SLIM_EINVAL;
        if (i && !(c.widths[i] > c.widths[i - 1])) return SLIM_EINVAL;
    }
    if (c.in_channels < 1 || c.in_channels > 4 || c.num_classes < 1 || c.num_classes > 1024 || c.max_batch < 1 ||
        !(c.bn_eps > 0.f) || (c.dtype != SLIM_BF16 && c.dtype != SLIM_FP32))
        return SLIM_EINVAL;
    if (c.image_hw < 16 || c.image_hw % 8) return SLIM_EUNSUPPORTED;
    if (c.norm != SLIM_NORM_BN && c.norm != SLIM_NORM_GN) return SLIM_EINVAL;
    if (c.norm == SLIM_NORM_GN) {   // groups must tile every active width (reading R16) and the 16-B vectors
        if (c.gn_group_channels < 8 || c.gn_group_channels % 8) return SLIM_EUNSUPPORTED;
        for (int s = 0; s < 4; ++s)
            for (int i = 0; i < c.n_widths; ++i)
                if (slim_channels(c.widths[i], c.base_channels[s]) % c.gn_group_channels) return SLIM_EUNSUPPORTED;
    }
    // BF16 stem/conv tiling: a 128-pixel tile is whole image rows and the stem's halo rows are 16-B multiples
    if (c.dtype == SLIM_BF16 && (c.image_hw > 32 || (c.image_hw * c.in_channels) % 8)) return SLIM_EUNSUPPORTED;
    for (int s = 0; s < 4; ++s) {
        if (c.blocks_per_seg[s] < 1 || c.blocks_per_seg[s] > 4) return SLIM_EINVAL;
        if (c.base_channels[s] < 16 || c.base_channels[s] > 1024) return SLIM_EINVAL;
        for (int i = 0; i < c.n_widths; ++i) {   // kernel channel counts (padded, see slim_act_channels)
            const int ch = slim_act_channels(c.widths[i], c.base_channels[s]);
            if (ch > c.base_channels[s]) return SLIM_EUNSUPPORTED;   // the padding must stay inside the weights
            if (s == 0 && ch > 64) return SLIM_EUNSUPPORTED;         // stem kernel holds <= 64 output channels
        }
    }
    slim_ctx *ctx = new slim_ctx();
    ctx->device = device;
    ctx->cfg = c;
    if (cudaSetDevice(device) != cudaSuccess) {
        delete ctx;
        return SLIM_ECUDA;
    }
    cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
        delete ctx;
        return SLIM_ECUDA;
    }
    ctx->encode = reinterpret_cast<PFN_encodeTiled>(fn);
    // internal workspace for slim_forward: max over segments at the widest width, B_max
    size_t ws = 0;
    for (int s = 0; s < 4; ++s) {
        const size_t b = seg_ws_bytes(c, s, c.widths[c.n_widths - 1], c.max_batch);
        ws = b > ws ? b : ws;
    }
    if (cudaMalloc(&ctx->ws, ws) != cudaSuccess) {
        cudaGetLastError();
        delete ctx;
        return SLIM_ENOMEM;
    }
    ctx->ws_bytes = ws;
    if (getenv("SLIM_CONV_TRACE")) cudaMalloc(&ctx->trace, 4096 * 8 * sizeof(unsigned long long));
    if (cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking) != cudaSuccess) {
        cudaFree(ctx->ws);
        delete ctx;
        return SLIM_ECUDA;
    }
    *out = ctx;
    return SLIM_OK;
}

void slim_destroy(slim_ctx *ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();
    clear_graphs(ctx);
    for (auto ev : ctx->prof_ev) cudaEventDestroy(ev);
    if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
    for (int s = 0; s < 4; ++s) free_segment(ctx->seg[s]);
    cudaFree(ctx->ws);
    delete ctx;
}

int slim_segment_loaded(const slim_ctx *ctx, int seg) {
    return ctx && seg >= 0 && seg < 4 && ctx->seg[seg].loaded ? 1 : 0;
}

slim_status slim_load_segment(slim_ctx *ctx, int seg, const slim_seg_weights *w, const slim_bn_set *bn) {
    if (!ctx) return SLIM_EINVAL;
    const slim_config &c = ctx->cfg;
    if (seg < 0 || seg > 3 || !w || !bn) return fail(ctx, SLIM_EINVAL, "load: bad arguments");
    LayerShape shp[kMaxLayers];
    const int n = segment_layers(c, seg, shp);
    if (w->n_conv != n) return fail(ctx, SLIM_EINVAL, "load: seg %d expects %d conv tensors, got %d", seg, n, w->n_conv);
    for (int l = 0; l < n; ++l)
        if (!w->conv_w[l]) return fail(ctx, SLIM_EINVAL, "load: conv_w[%d] is NULL", l);
    if (seg == 3 && (!w->fc_w || !w->fc_b)) return fail(ctx, SLIM_EINVAL, "load: seg 3 needs fc_w and fc_b");
    for (int i = 0; i < c.n_widths; ++i) {
        if (bn[i].n_layers != n || !bn[i].per_layer)
            return fail(ctx, SLIM_EINVAL, "load: BN set %d has %d layers, expected %d", i, bn[i].n_layers, n);
        for (int l = 0; l < n; ++l) {
            const slim_bn &b = bn[i].per_layer[l];
            if (!b.gamma || !b.beta || (c.norm == SLIM_NORM_BN && (!b.mean || !b.var)))
                return fail(ctx, SLIM_EINVAL, "load: BN arrays NULL");
        }
    }
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();   // no forward of this segment may be in flight (documented contract)
    clear_graphs(ctx);         // captured graphs hold the old weight addresses
    free_segment(ctx->seg[seg]);
    DevSegment &S = ctx->seg[seg];
    S.n_conv = n;
    const bool bf = c.dtype == SLIM_BF16;
    for (int l = 0; l < n; ++l) {
        DevLayer &L = S.L[l];
        L.sh = shp[l];
        const size_t cnt = static_cast<size_t>(L.sh.cout) * L.sh.k * L.sh.k * L.sh.cin;
        if (L.sh.is_stem || !bf) {   // CUDA-core kernels read fp32 (bf16-rounded in BF16 mode)
            std::vector<float> h(w->conv_w[l], w->conv_w[l] + cnt);
            if (bf)
                for (auto &v : h) v = bf_round(v);
            CUDA_TRY(ctx, cudaMalloc(&L.w, cnt * 4));
            CUDA_TRY(ctx, cudaMemcpy(L.w, h.data(), cnt * 4, cudaMemcpyHostToDevice));
            if (L.sh.is_stem && bf && L.sh.cout <= 64 && 9 * L.sh.cin <= 64) {
                // the stem's B operand as the kernel's shared-memory image: row co (K-major, 128 B) holds
                // w[co][k] for k < 9*c_img, 16-B piece j at (j ^ (co & 7)) (SWIZZLE_128B); rows >= c0 of a
                // width are never read (N = c0)
                std::vector<uint16_t> img(64 * 64, 0);
                const int K = 9 * L.sh.cin;
                for (int co = 0; co < L.sh.cout; ++co)
                    for (int k = 0; k < K; ++k)
                        img[co * 64 + (((k >> 3) ^ (co & 7)) << 3) + (k & 7)] = f2bf(h[static_cast<size_t>(co) * K + k]);
                CUDA_TRY(ctx, cudaMalloc(&L.stem_b, img.size() * 2));
                CUDA_TRY(ctx, cudaMemcpy(L.stem_b, img.data(), img.size() * 2, cudaMemcpyHostToDevice));
            }
        } else {
            std::vector<uint16_t> h(cnt);
            for (size_t i = 0; i < cnt; ++i) h[i] = f2bf(w->conv_w[l][i]);
            CUDA_TRY(ctx, cudaMalloc(&L.w, cnt * 2));
            CUDA_TRY(ctx, cudaMemcpy(L.w, h.data(), cnt * 2, cudaMemcpyHostToDevice));
        }
        // switchable BN, folded per width in fp64: s = gamma/sqrt(var+eps), t = beta - mean*s.
        // GN: the conv epilogue is the identity (s = 1, t = 0); gamma/beta go to the GN kernel.
        // Channels ch .. cp-1 (universal-width padding) get scale = shift = 0 (GN: gamma = beta = 0).
        for (int i = 0; i < c.n_widths; ++i) {
            const int ch = slim_channels(c.widths[i], L.sh.cout);
            const int cp = slim_act_channels(c.widths[i], L.sh.cout);
            const slim_bn &b = bn[i].per_layer[l];
            std::vector<float> sc(cp, 0.f), sh(cp, 0.f);
            for (int k = 0; k < ch; ++k) sc[k] = 1.f;
            if (c.norm == SLIM_NORM_GN) {
                std::vector<float> g(cp, 0.f), be(cp, 0.f);
                std::copy(b.gamma, b.gamma + ch, g.begin());
                std::copy(b.beta, b.beta + ch, be.begin());
                CUDA_TRY(ctx, cudaMalloc(&L.gn_gamma[i], cp * 4));
                CUDA_TRY(ctx, cudaMalloc(&L.gn_beta[i], cp * 4));
                CUDA_TRY(ctx, cudaMemcpy(L.gn_gamma[i], g.data(), cp * 4, cudaMemcpyHostToDevice));
                CUDA_TRY(ctx, cudaMemcpy(L.gn_beta[i], be.data(), cp * 4, cudaMemcpyHostToDevice));
            }
            for (int k = 0; k < ch && c.norm == SLIM_NORM_BN; ++k) {
                const double s = static_cast<double>(b.gamma[k]) /
                                 std::sqrt(static_cast<double>(b.var[k]) + static_cast<double>(c.bn_eps));
                sc[k] = static_cast<float>(s);
                sh[k] = static_cast<float>(static_cast<double>(b.beta[k]) - static_cast<double>(b.mean[k]) * s);
            }
            CUDA_TRY(ctx, cudaMalloc(&L.scale[i], cp * 4));
            CUDA_TRY(ctx, cudaMalloc(&L.shift[i], cp * 4));
            CUDA_TRY(ctx, cudaMemcpy(L.scale[i], sc.data(), cp * 4, cudaMemcpyHostToDevice));
            CUDA_TRY(ctx, cudaMemcpy(L.shift[i], sh.data(), cp * 4, cudaMemcpyHostToDevice));
        }
    }
    if (seg == 3) {
        const size_t fw = static_cast<size_t>(c.num_classes) * c.base_channels[3];
        CUDA_TRY(ctx, cudaMalloc(&S.fc_w, fw * 4));
        CUDA_TRY(ctx, cudaMalloc(&S.fc_b, c.num_classes * 4));
        CUDA_TRY(ctx, cudaMemcpy(S.fc_w, w->fc_w, fw * 4, cudaMemcpyHostToDevice));
        CUDA_TRY(ctx, cudaMemcpy(S.fc_b, w->fc_b, c.num_classes * 4, cudaMemcpyHostToDevice));
    }
    // fused-segment weight images (segments 1-3, narrow widths; kernels_fused.cu) for every (r_prev, r)
    // pair the fused kernel supports: built once here, so no first-use repack lands inside a graph capture
    if (seg > 0 && c.dtype == SLIM_BF16 && c.blocks_per_seg[seg] == 2 &&
        (c.norm == SLIM_NORM_BN || c.gn_group_channels == 16)) {
        for (int ri = 0; ri < c.n_widths; ++ri) {
            const int C = slim_channels(c.widths[ri], c.base_channels[seg]);
            if (C != slim_act_channels(c.widths[ri], c.base_channels[seg])) continue;
            for (int rp = 0; rp < c.n_widths; ++rp) {
                const int CI = slim_act_channels(c.widths[rp], c.base_channels[seg - 1]);
                if (!segn_fused_smem_bytes(seg, C, CI, c.norm == SLIM_NORM_GN)) continue;
                const size_t nb = segn_fused_image_bytes(seg, C, CI);
                CUDA_TRY(ctx, cudaMalloc(&S.fimg[rp][ri], nb));
                CUDA_TRY(ctx, cudaMemset(S.fimg[rp][ri], 0, nb));
                CUDA_TRY(ctx, build_segn_fused_image(S.fimg[rp][ri], S.L[0].w, S.L[1].w, S.L[2].w, S.L[3].w, S.L[4].w,
                                                     seg, C, CI, S.L[0].sh.cin, S.L[1].sh.cin, nullptr));
            }
        }
        CUDA_TRY(ctx, cudaDeviceSynchronize());
    }
    S.loaded = true;
    return SLIM_OK;
}

slim_status slim_unload_segment(slim_ctx *ctx, int seg) {
    if (!ctx || seg < 0 || seg > 3) return SLIM_EINVAL;
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();
    clear_graphs(ctx);
    free_segment(ctx->seg[seg]);
    return SLIM_OK;
}

size_t slim_segment_bytes(const slim_config *cfg, int seg, float r_prev, float r) {
    if (!cfg || seg < 0 || seg > 3) return 0;
    const slim_config &c = *cfg;
    if (width_index(c, r) < 0 || (seg > 0 && width_index(c, r_prev) < 0)) return 0;
    LayerShape shp[kMaxLayers];
    const int n = segment_layers(c, seg, shp);
    size_t bytes = 0;
    for (int l = 0; l < n; ++l) {
        const LayerShape &L = shp[l];
        const int co = slim_channels(r, L.cout);
        const int ci = L.is_stem ? L.cin : slim_channels(L.reads_prev ? r_prev : r, L.cin);
        const size_t eb = (L.is_stem || c.dtype == SLIM_FP32) ? 4 : 2;
        bytes += static_cast<size_t>(co) * L.k * L.k * ci * eb + 2 * static_cast<size_t>(co) * 4;
    }
    if (seg == 3) bytes += static_cast<size_t>(c.num_classes) * (slim_channels(r, c.base_channels[3]) + 1) * 4;
    return bytes;
}

size_t slim_forward_workspace_bytes(const slim_ctx *ctx, int seg, float, float r, int batch) {
    if (!ctx || seg < 0 || seg > 3 || batch < 1) return 0;
    return seg_ws_bytes(ctx->cfg, seg, r, batch);
}

slim_status slim_forward_ws(slim_ctx *ctx, int seg, float r_prev, float r, int batch, const void *in, void *out,
                            void *ws, size_t ws_bytes, void *stream) {
    int ri_prev, ri;
    slim_status s = validate_fwd(ctx, seg, r_prev, r, batch, in, out, &ri_prev, &ri);
    if (s) return s;
    if (!ws || !aligned16(ws) || ws_bytes < seg_ws_bytes(ctx->cfg, seg, r, batch))
        return fail(ctx, SLIM_EINVAL, "workspace too small or misaligned");
    if ((s = check_sticky(ctx))) return s;
    const std::string key = make_key('S', seg, ri_prev, ri, batch, in, static_cast<const void *>(out),
                                     static_cast<const void *>(ws));
    return run_graphed(ctx, key, static_cast<cudaStream_t>(stream), [&](cudaStream_t st) {
        return run_segment(ctx, seg, ri_prev, ri, batch, in, out, ws, st);
    });
}

slim_status slim_forward(slim_ctx *ctx, int seg, float r_prev, float r, int batch, const void *in, void *out,
                         void *stream) {
    if (!ctx) return SLIM_EINVAL;
    return slim_forward_ws(ctx, seg, r_prev, r, batch, in, out, ctx->ws, ctx->ws_bytes, stream);
}

size_t slim_chain_workspace_bytes(const slim_ctx *ctx, const float r[4], int batch) {
    if (!ctx || !r || batch < 1) return 0;
    size_t inter = 0, segws = 0;
    for (int s = 0; s < 4; ++s) {
        const size_t a = round256(act_bytes(ctx->cfg, s, r[s], batch));
        const size_t w = seg_ws_bytes(ctx->cfg, s, r[s], batch);
        inter = a > inter ? a : inter;
        segws = w > segws ? w : segws;
    }
    return 2 * inter + segws;
}

slim_status slim_forward_chain(slim_ctx *ctx, const float r[4], int batch, const void *in, float *logits, void *ws,
                               size_t ws_bytes, void *stream) {
    if (!ctx || !r) return SLIM_EINVAL;
    int rip[4], ri[4];
    slim_status s;
    for (int k = 0; k < 4; ++k)
        if ((s = validate_fwd(ctx, k, k ? r[k - 1] : r[0], r[k], batch, in, logits, &rip[k], &ri[k]))) return s;
    const size_t need = slim_chain_workspace_bytes(ctx, r, batch);
    if (!ws || !aligned16(ws) || ws_bytes < need) return fail(ctx, SLIM_EINVAL, "chain workspace too small");
    if ((s = check_sticky(ctx))) return s;
    size_t inter = 0;
    for (int k = 0; k < 4; ++k) {
        const size_t a = round256(act_bytes(ctx->cfg, k, r[k], batch));
        inter = a > inter ? a : inter;
    }
    char *o[2] = {static_cast<char *>(ws), static_cast<char *>(ws) + inter};
    char *segws = static_cast<char *>(ws) + 2 * inter;
    const std::string key = make_key('C', ri[0], ri[1], ri[2], ri[3], batch, in, static_cast<const void *>(logits),
                                     static_cast<const void *>(ws));
    return run_graphed(ctx, key, static_cast<cudaStream_t>(stream), [&](cudaStream_t st) {
        const void *cur = in;
        for (int k = 0; k < 4; ++k) {
            void *dst = (k == 3) ? static_cast<void *>(logits) : o[k & 1];
            slim_status s2 = run_segment(ctx, k, rip[k], ri[k], batch, cur, dst, segws, st);
            if (s2) return s2;
            cur = dst;
        }
        return SLIM_OK;
    });
}

slim_status slim_pack(const slim_config *cfg, const slim_request *q, int n, int B_max, slim_launch_desc *descs,
                      int max_descs, int *n_descs, uint32_t *order) {
    if (!cfg || n < 0 || B_max < 1 || !n_descs || (n > 0 && (!q || !descs || !order))) return SLIM_EINVAL;
    *n_descs = 0;
    const slim_config &c = *cfg;
    // key -> FIFO of request indices; a key is (seg, w_req idx, w_prev idx).  Buckets are one
    // flat array grouped by key (counting sort, stable: FIFO order inside a key).
    constexpr int kKeys = 4 * kMaxW * kMaxW;
    std::vector<int> key_of(n), bucket(n);
    int start[kKeys + 1] = {}, head[kKeys];
    for (int i = 0; i < n; ++i) {
        const int wr = width_index(c, q[i].w_req);
        const int wp = q[i].seg == 0 ? 0 : width_index(c, q[i].w_prev);
        if (q[i].seg < 0 || q[i].seg > 3 || wr < 0 || wp < 0) return SLIM_EINVAL;
        key_of[i] = (q[i].seg * kMaxW + wr) * kMaxW + wp;
        start[key_of[i] + 1]++;
    }
    for (int k = 0; k < kKeys; ++k) {
        start[k + 1] += start[k];
        head[k] = start[k];
    }
    for (int i = 0; i < n; ++i) bucket[head[key_of[i]]++] = i;
    for (int k = 0; k < kKeys; ++k) head[k] = start[k];   // consumed prefix of each bucket
    std::vector<char> taken(n, 0);
    int pos = 0, nd = 0;
    for (int i = 0; i < n; ++i) {   // Alg.1 LOOP: peek the FIFO head's key ...
        if (taken[i]) continue;
        if (nd >= max_descs) return SLIM_EINVAL;
        const int k = key_of[i];
        slim_launch_desc d;
        d.seg = q[i].seg;
        d.r = q[i].w_req;
        d.r_prev = q[i].seg == 0 ? q[i].w_req : q[i].w_prev;
        d.first = pos;
        d.batch = 0;
        while (head[k] < start[k + 1] && d.batch < B_max) {   // ... FORM-BATCH: up to B_max with that key, FIFO order
            const int j = bucket[head[k]++];
            taken[j] = 1;
            order[pos++] = static_cast<uint32_t>(j);
            d.batch++;
        }
        descs[nd++] = d;
    }
    *n_descs = nd;
    return SLIM_OK;
}

slim_status slim_gather(slim_ctx *ctx, const void *src, const uint32_t *idx, int n, size_t row_bytes, void *dst,
                        void *stream) {
    if (!ctx || n < 0 || (n > 0 && (!src || !idx || !dst)) || row_bytes % 16 || !aligned16(src) || !aligned16(dst))
        return ctx ? fail(ctx, SLIM_EINVAL, "gather: bad arguments") : SLIM_EINVAL;
    if (n == 0) return SLIM_OK;
    LaunchProf prof(ctx, static_cast<cudaStream_t>(stream));
    cudaError_t e = launch_gather(src, row_bytes, idx, n, row_bytes, dst, static_cast<cudaStream_t>(stream));
    prof.done(SLIM_K_GATHER, -1, -1, 0.f, 0.f, n, 0.0, 2.0 * n * static_cast<double>(row_bytes) + 4.0 * n);
    if (e != cudaSuccess) return fail(ctx, SLIM_ECUDA, "gather launch: %s", cudaGetErrorString(e));
    return SLIM_OK;
}

slim_status slim_scatter(slim_ctx *ctx, const void *src, const uint32_t *idx, int n, size_t row_bytes, void *dst,
                         size_t dst_stride, void *stream) {
    if (!ctx || n < 0 || (n > 0 && (!src || !idx || !dst)) || row_bytes % 16 || dst_stride % 16 || dst_stride < row_bytes ||
        !aligned16(src) || !aligned16(dst))
        return ctx ? fail(ctx, SLIM_EINVAL, "scatter: bad arguments") : SLIM_EINVAL;
    if (n == 0) return SLIM_OK;
    LaunchProf prof(ctx, static_cast<cudaStream_t>(stream));
    cudaError_t e = launch_scatter(src, idx, n, row_bytes, dst, dst_stride, static_cast<cudaStream_t>(stream));
    prof.done(SLIM_K_GATHER, -1, -1, 0.f, 0.f, n, 0.0, 2.0 * n * static_cast<double>(row_bytes) + 4.0 * n);
    if (e != cudaSuccess) return fail(ctx, SLIM_ECUDA, "scatter launch: %s", cudaGetErrorString(e));
    return SLIM_OK;
}

slim_status slim_launch(slim_ctx *ctx, const slim_launch_desc *d, const uint32_t *slots, const void *pool,
                        size_t pool_row_bytes, void *slab, void *out, void *ws, size_t ws_bytes, void *stream) {
    if (!ctx || !d) return SLIM_EINVAL;
    int ri_prev, ri;
    slim_status s = validate_fwd(ctx, d->seg, d->r_prev, d->r, d->batch, pool, out, &ri_prev, &ri);
    if (s) return s;
    const slim_config &c = ctx->cfg;
    const int Hin = d->seg == 0 ? c.image_hw : seg_hw(c, d->seg - 1);
    const int Cin = d->seg == 0 ? c.in_channels : slim_act_channels(d->r_prev, c.base_channels[d->seg - 1]);
    const size_t row = static_cast<size_t>(Hin) * Hin * Cin * elem_bytes(c);
    const void *in = pool;
    if (slots) {
        if (!slab || !aligned16(slab) || pool_row_bytes < row || pool_row_bytes % 16 || row % 16)
            return fail(ctx, SLIM_EINVAL, "launch: slab/pool rows invalid");
        LaunchProf prof(ctx, static_cast<cudaStream_t>(stream));
        cudaError_t e =
            launch_gather(pool, pool_row_bytes, slots, d->batch, row, slab, static_cast<cudaStream_t>(stream));
        prof.done(SLIM_K_GATHER, d->seg, -1, d->r_prev, d->r, d->batch, 0.0,
                  2.0 * d->batch * static_cast<double>(row) + 4.0 * d->batch);
        if (e != cudaSuccess) return fail(ctx, SLIM_ECUDA, "gather launch: %s", cudaGetErrorString(e));
        in = slab;
    }
    return slim_forward_ws(ctx, d->seg, d->r_prev, d->r, d->batch, in, out, ws, ws_bytes, stream);
}

slim_status slim_set_sm_share(slim_ctx *ctx, float r, float share) {
    if (!ctx) return SLIM_EINVAL;
    const int ri = width_index(ctx->cfg, r);
    if (ri < 0 || !(share > 0.f && share <= 1.f)) return fail(ctx, SLIM_EINVAL, "sm_share: bad width or share");
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();   // captured graphs bake the grid sizes: drop them once nothing is in flight
    clear_graphs(ctx);
    ctx->sm_share[ri] = share;
    return SLIM_OK;
}

slim_status slim_set_graph_mode(slim_ctx *ctx, int enable) {
    if (!ctx) return SLIM_EINVAL;
    if (!enable) clear_graphs(ctx);
    ctx->graph_mode = enable != 0;
    return SLIM_OK;
}

slim_status slim_profile_begin(slim_ctx *ctx, int max_launches) {
    if (!ctx || max_launches < 1) return SLIM_EINVAL;
    cudaSetDevice(ctx->device);
    while (ctx->prof_ev.size() < 2 * static_cast<size_t>(max_launches)) {
        cudaEvent_t ev;
        CUDA_TRY(ctx, cudaEventCreate(&ev));
        ctx->prof_ev.push_back(ev);
    }
    ctx->prof_rec.clear();
    ctx->prof_rec.reserve(max_launches);
    ctx->prof_on = true;
    return SLIM_OK;
}

slim_status slim_profile_end(slim_ctx *ctx, slim_profile_record *out, int max_out, int *n_out) {
    if (!ctx || !n_out) return SLIM_EINVAL;
    ctx->prof_on = false;
    CUDA_TRY(ctx, cudaDeviceSynchronize());
    int n = 0;
    for (size_t i = 0; i < ctx->prof_rec.size() && n < max_out; ++i, ++n) {
        float ms = 0.f;
        CUDA_TRY(ctx, cudaEventElapsedTime(&ms, ctx->prof_ev[2 * i], ctx->prof_ev[2 * i + 1]));
        ctx->prof_rec[i].ms = ms;
        if (out) out[n] = ctx->prof_rec[i];
    }
    *n_out = out ? n : static_cast<int>(ctx->prof_rec.size());
    return SLIM_OK;
}

slim_status slim_last_error(slim_ctx *ctx) {
    if (!ctx) return SLIM_EINVAL;
    return check_sticky(ctx);
}
const char *slim_last_error_msg(const slim_ctx *ctx) { return ctx ? ctx->msg.c_str() : "no context"; }
uint64_t slim_launch_count(const slim_ctx *ctx) { return ctx ? ctx->launches.load() : 0; }
int slim_num_sms(const slim_ctx *ctx) { return ctx ? ctx->num_sms : 0; }
// diagnostics (not in slim.h): copy the per-CTA timestamps of the last traced conv launch
SLIM_API int slimdbg_trace(slim_ctx *ctx, unsigned long long *host, int n) {
    if (!ctx || !ctx->trace) return -1;
    cudaDeviceSynchronize();
    return cudaMemcpy(host, ctx->trace, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : -1;
}

}  // extern "C"
