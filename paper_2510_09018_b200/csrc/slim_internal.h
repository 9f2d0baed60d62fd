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
constexpr int kConvThreads = 192;  // warp0 TMA, warp1 MMA (+TMEM alloc), warps2-5 epilogue
constexpr int kMaxStages = 8;

enum EpiMode : int {
    EPI_BN_RELU = 0,        // relu(s*acc + t)                       (stem-less conv1, K1)
    EPI_BN_ADD_RELU = 1,    // relu(s*acc + t + residual)            (conv2, identity shortcut, K2)
    EPI_BN_PROJ_RELU = 2,   // relu(s*acc + t + s_sc*acc_sc + t_sc)  (conv2 + 1x1 projection, K3)
};

struct GemmPart {          // one GEMM accumulated into one TMEM accumulator
    int ksize, stride, pad;
    int c_in;              // active input channels (TMA bound: channels >= c_in read as 0)
    int n_chunks;          // ceil(c_in / 64)
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
    uint32_t stage_b_bytes;   // n_tile * 128
    uint32_t n_out_chunks;    // ceil(n_tile / 64) staging buffers of 16 KiB
};

size_t conv_umma_smem_bytes(const ConvArgs &a);
cudaError_t launch_conv_umma(const ConvArgs &a, const CUtensorMap &tmA0, const CUtensorMap &tmB0,
                             const CUtensorMap &tmA1, const CUtensorMap &tmB1, const CUtensorMap &tmRes,
                             const CUtensorMap &tmOut, int grid, cudaStream_t stream);
int conv_umma_max_ctas_per_sm(size_t smem_bytes);

// ---- CUDA-core kernels (kernels_simt.cu) ------------------------------------
cudaError_t launch_stem_bf16(const uint16_t *in, const float *w, int cin_full, const float *scale,
                             const float *shift, uint16_t *out, int B, int H, int W, int cimg, int c0,
                             cudaStream_t s);
cudaError_t launch_head_bf16(const uint16_t *in, const float *fc_w, const float *fc_b, float *logits,
                             int B, int P, int c3, int c3_full, int K, cudaStream_t s);
// dst row i (row_bytes, multiple of 16) = src + idx[i]*src_stride (bytes)
cudaError_t launch_gather(const void *src, size_t src_stride, const uint32_t *idx, int n, size_t row_bytes,
                          void *dst, cudaStream_t s);

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
};
cudaError_t launch_conv_f32(const ConvF32Args &a, cudaStream_t s);
cudaError_t launch_stem_f32(const float *in, const float *w, int cin_full, const float *scale,
                            const float *shift, float *out, int B, int H, int W, int cimg, int c0,
                            cudaStream_t s);
cudaError_t launch_head_f32(const float *in, const float *fc_w, const float *fc_b, float *logits,
                            int B, int P, int c3, int c3_full, int K, cudaStream_t s);

}  // namespace slim
