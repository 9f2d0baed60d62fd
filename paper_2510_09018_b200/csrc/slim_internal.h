// slim_internal.h -- private declarations shared by the libslim.so sources.
// Not part of the ABI (include/slim.h is).  Nothing here is visible to oracle/.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>

namespace slim {

// ---- implicit-GEMM conv on tcgen05 (kernels_umma.cu) -----------------------
// GEMM view of a conv: M = B*Ho*Wo output pixels (NHWC order),
// N = c_out, K = k*k*c_in.  One CTA tile is 128 pixels x n_tile channels.
constexpr int kTileM = 128;        // UMMA M (cta_group::1): TMEM lane = tile row
constexpr int kChunk = 64;         // channels per K-block = one 128-byte SW128 row
constexpr int kTileABytes = kTileM * kChunk * 2;   // 16 KiB A operand per K-block
constexpr int kConvThreads = 448;  // warps 0,2,12,13 TMA producers, warp1 MMA (+TMEM alloc), warp3 residual TMA,
                                   // warps4-11 epilogue
constexpr int kMaxStages = 8;
constexpr int kEpiWarp0 = 4;       // first epilogue warp (warp 3 idles)
constexpr int kEpiThreads = 256;   // 8 epilogue warps, two per TMEM lane quarter

enum EpiMode : int {
    EPI_BN_RELU = 0,        // relu(s*acc + t)                       (stem-less conv1, K1)
    EPI_BN_ADD_RELU = 1,    // relu(s*acc + t + residual)            (conv2, identity shortcut, K2)
    EPI_BN_PROJ_RELU = 2,   // relu(s*acc + t + s_sc*acc_sc + t_sc)  (conv2 + 1x1 projection, K3)
};

struct GemmPart {          // one GEMM accumulated into one TMEM accumulator
    int ksize, stride, pad;
    int c_in;              // active input channels (TMA bound: channels >= c_in read as 0)
    int ck;                // channels per K-block chunk: 16 | 32 (exact narrow boxes) | 64
    int rbk;               // operand row bytes = 2*ck = the swizzle span (32 | 64 | 128 B)
    int n_chunks;          // ceil(c_in / ck)
    int n_kblocks;         // ksize*ksize*n_chunks
};

struct ConvArgs {
    int B, Ho, Wo;
    int tile_imgs, tile_rows, tiles_per_img;   // tile = tile_imgs x tile_rows x Wo = 128 pixels
    int m_tiles, n_tiles, n_tile, c_out;
    int n_parts;
    GemmPart part[2];
    int epi;
    const float *scale0, *shift0, *scale1, *shift1;   // folded BN of the two accumulators
    int n_stages, acc_stages, acc_stride, tmem_cols;
    uint32_t a_tile_bytes;    // 128 * max part rbk (one A stage)
    uint32_t stage_b_bytes;   // n_tile * max part rbk, rounded up to 1 KiB
    int co_chunk, rbo;        // output channels per staging chunk (16 | 32 | 64) and its row bytes
    uint32_t n_out_chunks;    // ceil(n_tile / co_chunk) staging chunks of 128*rbo bytes
    int res_slots;            // residual prefetch ring depth (EPI_BN_ADD_RELU), 1 or 2
    int n_prod;               // TMA producer warps (1..4); k-block kb is loaded by producer kb % n_prod
    int mc;                   // cluster size along N (1 = no cluster): the mc CTAs of a cluster compute the
                              // same M tile for different N tiles; each k-block's A box is loaded once and
                              // TMA-multicast to all of them
    // fused global-average-pool (last conv of the network): instead of storing the
    // [B,Ho,Wo,c_out] tile, average each image's Ho*Wo rows and write fp32 pooled[B][c_out]
    float *pool_out;          // nullptr = normal store
    int debug;                // diagnostics only (env SLIM_CONV_DEBUG): 1 = no TMA loads, 2 = no MMAs
    unsigned long long *trace;   // diagnostics only (env SLIM_CONV_TRACE): per-CTA %globaltimer stamps
    float relu_lo;            // output = max(v, relu_lo): 0 = ReLU; -inf = raw (GroupNorm mode, pre-norm output)
};

size_t conv_umma_smem_bytes(const ConvArgs &a);

// split-K conv over a thread-block cluster with a DSMEM reduction (kernels_splitk.cu)
struct SplitArgs {
    int B, Ho, Wo;
    int tile_imgs, tile_rows, tiles_per_img, m_tiles;
    int n_tile, c_out;        // output tile 128 x n_tile (n_tile | c_out, <= 256, n_parts*n_tile <= 512)
    int n_parts;
    GemmPart part[2];         // 64-channel chunks (ck = 64, 128-B rows) for both parts
    int epi;
    const float *scale0, *shift0, *scale1, *shift1;
    int ks;                   // K splits = cluster size (2..8); CTA r of a cluster takes k-blocks [r*G/ks, (r+1)*G/ks)
    int w_o;                  // output channels each CTA finishes: n_tile / ks (multiple of 16)
    int co_chunk, rbo;        // staging chunk of the owner slice (16 | 32 | 64 channels) and its row bytes
    uint32_t n_out_chunks;    // w_o / co_chunk
    int n_stages;
    uint32_t stage_bytes;     // A 16 KiB + B n_tile*128 B; the drained stages hold the DSMEM receive buffer
    int n_prod, tmem_cols;
    float *pool_out;
    float relu_lo;            // 0 = ReLU, -inf = raw pre-norm output (GroupNorm mode)
};
size_t conv_splitk_smem_bytes(const SplitArgs &a);
size_t conv_splitk_recv_bytes(const SplitArgs &a);
cudaError_t launch_conv_splitk(const SplitArgs &a, const CUtensorMap &tmA0, const CUtensorMap &tmB0,
                               const CUtensorMap &tmA1, const CUtensorMap &tmB1, const CUtensorMap &tmRes,
                               const CUtensorMap &tmOut, int grid, cudaStream_t stream, bool pdl);

// stride-1 3x3 conv, one halo box per channel chunk + kw-split accumulators (kernels_halo.cu)
struct HaloArgs {
    int B, H, W;              // output = input spatial size (stride 1, pad 1)
    int rows, tiles_per_img;  // tile = rows full image rows of tile_imgs images, rows*W*tile_imgs = 128
    int tile_imgs, row_px;    // images per tile (1 unless H*W < 128); pixels per halo row = tile_imgs*W
    int m_tiles, n_tiles, n_tile, c_out, c_in, n_chunks;
    int epi;                  // EPI_BN_RELU, EPI_BN_ADD_RELU or EPI_BN_PROJ_RELU (1x1 stride-2 shortcut)
    const float *scale, *shift;
    const float *scale1, *shift1;   // projection BN (EPI_BN_PROJ_RELU)
    int c_in_p, n_chunks_p;   // projection input channels and 64-channel chunks
    float *pool_out;          // fused average pool -> fp32 [B][c_out] (rows == 4, row_px == 32), else nullptr
    int stride2;              // stride-2 conv: input [B, 2H, 2W, c_in] as parity planes (tmA even rows, tmA1 odd)
    int small;                // compact variant: 8 epilogue warps, two CTAs per SM (narrow layers)
    int x3;                   // 1: three kw-shifted halo boxes per chunk, one accumulator; 2: two boxes, two
                              // accumulators (a_bytes = one box)
    int stationary;           // all weights resident in smem (one B slot of n_chunks*9 taps)
    int sa, sb;               // A ring slots (one per chunk), B ring slots (one per (chunk, kh)) -- each <= 4
    int acc_stride, acc_stages, tmem_cols;
    int ck, rbk;              // input channels per chunk (16 | 32 | 64) and operand row bytes
    int co_chunk, rbo;        // output channels per staging chunk and its row bytes
    uint32_t a_bytes, b_bytes;   // halo box bytes (expect_tx), B slot bytes
    uint32_t a_slot;             // A ring slot stride (>= a_bytes; a projection chunk also fits)
    uint32_t n_out_chunks;
    int res_slots;
    int kw_fuse;              // kw taps per MMA (1..3): their accumulators are adjacent (acc_stride = n_tile)
    int stage_cols;           // TMEM columns per accumulator stage (3 kw accumulators, 32-aligned)
    int epi_groups;           // 2: epilogue warps 4-7 / 8-11 take even / odd tiles; 1: they split columns
    int debug;
    unsigned long long *trace;
    float relu_lo;            // 0 = ReLU, -inf = raw pre-norm output (GroupNorm mode)
    // GroupNorm mode: per-(image, tile, 16-channel group) statistics of the stored (bf16) raw output,
    // (mean, M2) over the tile's pixels of that image, at gn_part[(n*tiles_per_img + ti)*(c_out/16) + g];
    // nullptr = off.  The GN apply kernel then merges them (launch_gn_apply_part).
    float2 *gn_part;
    // streamed-weight multicast: a cluster of bmc CTAs (1 = off) works on bmc consecutive M tiles of one
    // N tile; each CTA loads 1/bmc of every B stage (rows rank*n_tile/bmc.., tmBh: box [ck, n_tile/bmc, 1])
    // and multicasts it to all, so the cluster reads each weight byte from L2 once instead of bmc times
    int bmc;
    // 2-SM MMA (cta_group::2): a CTA pair (cluster of 2) on consecutive M tiles of one N tile issues ONE
    // M = 256 MMA from the even CTA; each CTA loads its own A tile and HALF of every B stage (1.5 n_tile
    // rows, tmBh: box [ck, n_tile/2, 1]), so the pair pulls each weight byte from L2 once and each SM
    // ingests half of it.  Needs streamed B, kw_fuse == 3, bmc == 1.
    int pair;
    // GroupNorm in the epilogue (GN mode): tiles that cover whole images (tiles_per_img == 1,
    // segments 2-3) reduce each (image, 16-channel group)'s statistics from the fp32 accumulators and
    // normalise with scale = gamma, shift = beta (scale1 / shift1: the projection's); relu_lo = 0
    int gn_fuse;
    float gn_eps;
    int gn_pairs;   // GN with two M tiles per image (segment 1): one CTA takes both (acc_stages 2, one tile group)
    // Tile-granular dependencies between consecutive halo convs of a segment (same M tiling) instead of
    // waiting for the whole previous grid (griddepcontrol.wait): flag_in[mt] counts the previous layer's
    // finished (mt, any N tile) tiles; a tile waits until its input M tiles (mt-1..mt+1 of the same image,
    // or mt for whole-image tiles) reach flag_in_target (= that layer's n_tiles).  flag_out: this layer's
    // counters (one red.release per finished tile, after its TMA store completed).  flag_zero: counters
    // of later layers this kernel clears (after its own griddepcontrol.wait, before it lets dependents
    // launch).  All nullptr = the plain PDL dependency.
    int nfast;   // N-fastest tile order (the N tiles of an M tile on neighbouring CTAs); 0 = M-fastest
    uint32_t *flag_in, *flag_out, *flag_zero;
    int flag_in_target, flag_zero_n;
};
constexpr int kMaxSB = 8;                    // halo kernel: B ring slots (barrier pairs) at most
constexpr int kHaloBars = 24 + 2 * kMaxSB;   // a_full/empty[4] b_full/empty[kMaxSB] t_full/empty[4] r_full/empty[4]
size_t conv_halo_smem_bytes(const HaloArgs &a);
cudaError_t launch_conv_halo(const HaloArgs &a, const CUtensorMap &tmA, const CUtensorMap &tmB,
                             const CUtensorMap &tmRes, const CUtensorMap &tmOut, const CUtensorMap &tmA1,
                             const CUtensorMap &tmB1, const CUtensorMap &tmBh, int grid, cudaStream_t stream, bool pdl);
cudaError_t launch_conv_umma(const ConvArgs &a, const CUtensorMap &tmA0, const CUtensorMap &tmB0,
                             const CUtensorMap &tmA1, const CUtensorMap &tmB1, const CUtensorMap &tmRes,
                             const CUtensorMap &tmOut, int grid, cudaStream_t stream, bool pdl);
int conv_umma_max_ctas_per_sm(size_t smem_bytes);

// stem (conv3x3 c_img -> c0 + BN + ReLU) on tcgen05, A built in smem (kernels_umma.cu)
struct StemArgs {
    const uint16_t *in;            // [B][H][W][cimg] bf16
    const float *w;                // [c0_full][9*cimg] fp32 (bf16-representable), rows >= c0 unread
    const void *b_img;             // the same weights as the kernel's SW128 bf16 B tile (8 KiB, built at load)
    int w_stride;                  // 9*cimg_full
    const float *scale, *shift;    // folded BN at this width, c0 entries
    int B, H, W, cimg, c0;
    int tile_rows, m_tiles, tmem_cols;
    unsigned long long *trace;     // diagnostics only (SLIM_CONV_TRACE): CTA 0 role x tile %globaltimer stamps
    float relu_lo;                 // 0 = ReLU, -inf = raw pre-norm output (GroupNorm mode)
};
// (kernels_stem.cu) tmIn: the image as a 3-D map (W*cimg, H, B), box (W*cimg, tile_rows+2, 1), no swizzle
cudaError_t launch_stem_umma(const StemArgs &a, const CUtensorMap &tmIn, const CUtensorMap &tmOut, int grid,
                             cudaStream_t stream, bool pdl);

// ---- segment 0 as one kernel for the narrow widths (kernels_fused.cu) ----------------------
// stem + two BasicBlocks, one image per CTA, activations resident in shared memory; c0 = 16 | 32
struct FusedSeg0Args {
    const uint16_t *in;            // images [B][32][32][3] bf16
    uint16_t *out;                 // segment output [B][32][32][c0] bf16
    int B, c0, cin_full;           // cin_full: the convs' full input width (weight row stride)
    const uint16_t *w[4];          // the four convs' full-width KRSC bf16 weights (manifest order)
    const void *stem_b;            // the stem's SW128 B image (64 rows x 128 B, K = 27 zero-padded)
    const float *scale[5], *shift[5];   // folded BN of stem + four convs at this width, c0 entries
    unsigned long long *trace;     // diagnostics only (SLIM_CONV_TRACE): CTA 0 phase %globaltimer stamps
    int cluster;                   // CTAs per image: 1 (whole image per CTA) or 8 (one 4-row tile each, DSMEM halo)
    int gn;                        // GroupNorm (16-channel groups): scale / shift carry gamma / beta
    float eps;
};
size_t seg0_fused_smem_bytes(int c0, int P);

// segments 1-3 as one kernel for the narrow widths (kernels_fused.cu): units of G images (seg 1: 1, 2: 2,
// 3: 8), activations in shared memory, weights streamed from a pre-swizzled image (build_segn_fused_image)
struct FusedSegArgs {
    const uint16_t *in;            // previous segment's output [B][2H][2W][CI] bf16
    uint16_t *out;                 // [B][H][W][C] bf16 (segments 1, 2)
    float *pool_out;               // segment 3: fp32 [B][C] average pool (the FC follows), else nullptr
    int B, CI;
    const uint8_t *wimg;           // the weight image of this (segment, r_prev, r)
    const float *scale[5], *shift[5];   // folded BN: b0c1, b0c2, projection, b1c1, b1c2 (C entries)
    uint32_t smem_budget;          // dynamic smem the launch reserved (the ring takes what is left)
    size_t wimg_rank_bytes;        // one cluster rank's part of the image (set by launch_segn_fused)
    int gn;                        // GroupNorm (16-channel groups): scale / shift carry gamma / beta
    float eps;
    unsigned long long *trace;     // diagnostics only (SLIM_CONV_TRACE): CTA 0 phase %globaltimer stamps
};
int segn_fused_cluster(int seg, int C);                 // CTAs per unit (output channels split over them)
size_t segn_fused_smem_bytes(int seg, int C, int CI, bool gn = false);   // 0 = unsupported / does not fit
size_t segn_fused_image_bytes(int seg, int C, int CI);
cudaError_t build_segn_fused_image(void *img, const void *w0, const void *w1, const void *wp, const void *w3,
                                   const void *w4, int seg, int C, int CI, int cin0_full, int cf_full, cudaStream_t st);
// units_grid: clusters (units in flight); the grid is units_grid * segn_fused_cluster(seg, C) CTAs
cudaError_t launch_segn_fused(const FusedSegArgs &a, int seg, int C, int units_grid, cudaStream_t stream, bool pdl);
cudaError_t launch_seg0_fused(const FusedSeg0Args &a, int grid, cudaStream_t stream, bool pdl);

// ---- CUDA-core kernels (kernels_simt.cu) ------------------------------------
cudaError_t launch_stem_bf16(const uint16_t *in, const float *w, int cin_full, const float *scale,
                             const float *shift, uint16_t *out, int B, int H, int W, int cimg, int c0,
                             cudaStream_t s, float relu_lo = 0.f);
cudaError_t launch_head_bf16(const uint16_t *in, const float *fc_w, const float *fc_b, float *logits,
                             int B, int P, int c3, int c3_full, int K, cudaStream_t s, bool pdl);
// FC head on pooled fp32 features [B][c3] (pool fused into the last conv)
cudaError_t launch_fc_f32(const float *pooled, const float *fc_w, const float *fc_b, float *logits, int B, int c3,
                          int c3_full, int K, cudaStream_t s, bool pdl);
// dst row i (row_bytes, multiple of 16) = src + idx[i]*src_stride (bytes)
cudaError_t launch_gather(const void *src, size_t src_stride, const uint32_t *idx, int n, size_t row_bytes,
                          void *dst, cudaStream_t s);

// dst + idx[i]*dst_stride (bytes) <- src row i (row_bytes, multiple of 16)
cudaError_t launch_scatter(const void *src, const uint32_t *idx, int n, size_t row_bytes, void *dst, size_t dst_stride,
                           cudaStream_t s);

// FP32 mode (TF32 off): SIMT direct conv with the same fused epilogues.
struct ConvF32Args {
    const float *x;  int B, H, W, c_in;          // part 0 input, dense NHWC
    const float *w;  int cin_full, k, stride, pad;
    const float *x1; int H1, W1, c_in1, stride1; // projection input (EPI_BN_PROJ_RELU), 1x1 pad 0
    const float *w1; int cin1_full;
    const float *res;                            // residual (EPI_BN_ADD_RELU), shape of out
    const float *scale0, *shift0, *scale1, *shift1;
    float *out; int Ho, Wo, c_out;
    int epi;
    float relu_lo;                               // 0 = ReLU, -inf = raw pre-norm output (GroupNorm mode)
    int max_ctas;                                // persistent-grid cap of the GEMM kernels (0 = one CTA per tile)
    // split-K (layers without a projection whose tiles leave most SMs idle): ksplit CTAs per tile take
    // consecutive ranges of the K steps and write raw fp32 partials part[split][pixel][c_out]; a reduce
    // kernel sums them in split order (deterministic) and applies the epilogue.  ksplit depends on the
    // layer shape and max_batch only (never on B), so the summation order is batch independent.
    int ksplit;
    float *part;
};
cudaError_t launch_conv_f32(const ConvF32Args &a, cudaStream_t s);
cudaError_t launch_stem_f32(const float *in, const float *w, int cin_full, const float *scale,
                            const float *shift, float *out, int B, int H, int W, int cimg, int c0,
                            cudaStream_t s, float relu_lo = 0.f);
cudaError_t launch_head_f32(const float *in, const float *fc_w, const float *fc_b, float *logits,
                            int B, int P, int c3, int c3_full, int K, cudaStream_t s, bool pdl);

// ---- GroupNorm variant (kernels_gn.cu, reading R16) ---------------
struct GnArgs {
    const void *y;                 // raw conv output [B][HW][C] (bf16 or fp32)
    const void *yp;                // raw projection-shortcut output (same shape) or nullptr
    const void *res;               // identity residual (same shape) or nullptr
    const float *gamma, *beta;     // GN affine of this width, C entries
    const float *gamma_p, *beta_p; // the shortcut's GN affine (yp != nullptr)
    void *out;                     // may alias y
    int B, HW, C, cpg, gpc;        // cpg channels per group; gpc groups per CTA (divides C/cpg)
    float eps, relu_lo;            // relu_lo 0 = ReLU, -inf = none
    int max_ctas;                  // persistent-grid cap (0 = one CTA per (image, slice))
    float *pool_out;               // != nullptr: write the average pool fp32 [B][C] instead of out
};
int gn_groups_per_cta(int B, int HW, int C, int cpg, bool fp32);
cudaError_t launch_gn(const GnArgs &a, bool fp32, cudaStream_t s, bool pdl);
// GN apply from statistics partials the producing conv wrote (HaloArgs::gn_part): no reduction over
// the image here -- an elementwise pass: out = act(GN(y) [+ res]) (bf16), or the average pool.
struct GnPartArgs {
    const uint16_t *y;             // raw conv output [B][HW][C] bf16
    const float2 *part;            // (mean, M2) per (image, tile, 16-channel group), tiles_per_img per image
    const uint16_t *res;           // identity residual or nullptr
    const float *gamma, *beta;     // GN affine, C entries
    uint16_t *out;                 // may alias y
    float *pool_out;               // != nullptr: fp32 [B][C] average pool instead of out
    int B, HW, C, tiles_per_img;
    float part_count;              // values per partial (pixels of the image in one tile x 16)
    float eps, relu_lo;
    int max_ctas;
};
cudaError_t launch_gn_apply_part(const GnPartArgs &a, cudaStream_t s, bool pdl);

}  // namespace slim
