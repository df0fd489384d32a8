// Persistent warp-specialised tcgen05 GEMM: D[M,N] = A[M,K] . B[N,K]^T (both K-major bf16), FP32
// accumulation in TMEM, TMA loads through an mbarrier ring, fused epilogues for the PrefillOnly layer:
//   EPI_BF16       plain bf16 store                      (generic)
//   EPI_RESID_F32  resid[m,n] += acc (fp32, in place)    (O-proj and down-proj + residual)
//   EPI_SILU_MUL   act = silu(gate) * up, gate/up interleaved in 16-column groups (ps/numerics.py:123-124,168)
//   EPI_QKV_ROPE   RoPE (rotate-half, per 128-wide head) on q/k columns, bf16 store of the qkv row
//   EPI_F32        plain fp32 store                      (tests / LM head)
#pragma once
#include "sm100.cuh"

namespace po {

enum GemmEpi : int { EPI_BF16 = 0, EPI_RESID_F32 = 1, EPI_SILU_MUL = 2, EPI_QKV_ROPE = 3, EPI_F32 = 4 };

struct GemmArgs {
  int M, N, K;
  int a_row0;           // first row of A addressed through the A tensor map (chunked MLP)
  void* out;            // bf16 or fp32 output (EPI_BF16 / EPI_SILU_MUL / EPI_QKV_ROPE / EPI_F32)
  long long ldo;        // elements
  float* resid;         // EPI_RESID_F32
  long long ldr;
  const float2* rope;   // [pos][64] (cos, sin) for EPI_QKV_ROPE
  int pos_offset;       // absolute position of row 0
  int rope_cols;        // columns [0, rope_cols) are rotated (q and k heads)
  const float* bias;    // EPI_QKV_ROPE: optional per-column bias added before RoPE (Qwen2 q/k/v bias)
  // Fused RMSNorm (the norm is folded across the GEMM: (x/rms . g) W^T = (1/rms) ((x . g) W^T)):
  //  consumer side (EPI_QKV_ROPE, EPI_SILU_MUL): A holds bf16(x . g); the epilogue scales each output row by
  //    rsqrt(sum_seg ss_in[row][seg] / norm_dim + eps) before bias / RoPE / SiLU.
  //  producer side (EPI_RESID_F32): after resid += acc, also write xg_out[row][col] = bf16(resid . g_next[col])
  //    and ss_out[row][seg] = sum of resid^2 over 128-column segment seg (two per 256-column tile).
  const float* ss_in;
  int ss_nseg;          // 128-column segments per row (= hidden / 128)
  float norm_eps;
  int norm_dim;
  __nv_bfloat16* xg_out;
  long long ldxg;
  const float* g_next;
  float* ss_out;
  // split-K (small-M GEMMs, e.g. prefix-hit requests): k_splits > 1 writes fp32 partials to `split_ws`
  // ([k_splits][M][N]) and a reduce kernel applies the epilogue after summing in a fixed order.
  int k_splits;
  int kb_per_split;
  float* split_ws;
  size_t split_ws_bytes;  // capacity of split_ws; a launch whose split needs more runs unsplit
  // EPI_QKV_ROPE prefix-pool admission (replaces a separate scatter pass): rows whose 16-token block b (absolute
  // position / 16) has kv_slot[b] >= 0 also store their K/V columns [kv_col0, kv_col0 + kv_dim) into
  // kv_pool[(slot * pool_layers + pool_layer) * 16 + position % 16][kv_dim].
  const int* kv_slot;
  __nv_bfloat16* kv_pool;
  int pool_layers, pool_layer, kv_col0, kv_dim;
  // FP8 (W8A8, E4M3 operands; gemm_launch_pair_f8 only): acc[m,n] is dequantised as acc * a_scale[m] * b_scale[n]
  // (per-row activation scale from quantize_rows_e4m3, per-output-channel weight scale) before the epilogue.
  const float* a_scale;
  const float* b_scale;
  // Stream-K swap-AB kernel (gemm_sk.cu, M <= 256): fp32 partial slots [num_sms][2][256][128] and one flag per slot
  // (128-byte stride); a launch raises its dump flags to sk_epoch, which must grow from launch to launch.
  float* sk_ws;
  uint32_t* sk_flags;
  uint32_t sk_epoch;
  // tile raster of the row-major kernels: m-blocks per sweep over N (0 = the launcher's choice by K)
  int group_m;
  // stream-K + reduce (gemm_sk.cu, sk_red = 1, opt-in PO_SK_RED=1): every segment's partial goes to split_ws slice j
  // (its contributor index within the tile, k order) and splitk_reduce_kernel sums each tile's contributors of the
  // equal-range stream-K split (sk_w work items, sk_p pairs, sk_nk k-blocks per tile)
  int sk_red;
  int sk_p, sk_nk;
  long long sk_w;
};

struct GemmPlan {
  const void* A;       // activation base and leading dimension (the swap-AB kernel builds its own map over it)
  long long lda;
  CUtensorMap map_a;
  CUtensorMap map_b;   // 256-row boxes (1-CTA kernel)
  CUtensorMap map_b2;  // 128-row boxes (2-CTA pair kernel, 256 x 256 tiles)
  CUtensorMap map_b3;  // 64-row boxes (2-CTA pair kernel, 256 x 128 tiles for small M)
  int M, N, K;
};

// Host helpers (gemm.cu)
int make_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t row_stride_bytes,
                      uint32_t box_inner, uint32_t box_outer);
// 3-D map (d0 innermost, 128B swizzle), e.g. the prefix pool [slot*layer][block_tokens][kv_dim].
int make_tmap_3d_bf16(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t stride1_bytes,
                      uint64_t stride2_bytes, uint32_t b0, uint32_t b1, uint32_t b2);
int make_tmap_4d_bf16(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t d3,
                      uint64_t stride1_bytes, uint64_t stride2_bytes, uint64_t stride3_bytes, uint32_t b0, uint32_t b1,
                      uint32_t b2, uint32_t b3);
int make_tmap_2d_epi(CUtensorMap* map, const void* base, bool f32, uint64_t cols, uint64_t rows, uint64_t row_stride_bytes,
                     bool swizzle128);
int make_tmap_store_3d(CUtensorMap* map, const void* base, bool f32, uint64_t d0, uint64_t d1, uint64_t d2,
                       uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t b0, uint32_t b1);
int gemm_plan(GemmPlan* plan, const void* A, long long lda, const void* B, long long ldb, int M, int N, int K);
int gemm_run(const GemmPlan& plan, int epi, const GemmArgs& args, cudaStream_t stream);
// A/B maps built once (weights at init, activation buffers at init with their max rows).
int gemm_launch(const CUtensorMap& map_a, const CUtensorMap& map_b, int epi, const GemmArgs& args,
                cudaStream_t stream);
// Workspace bytes a launch of this shape needs for split-K (0 = no split).
size_t gemm_split_ws_bytes(int M, int N, int K);
// 2-CTA pair variant (M > 128): map_b2 must be built with 128-row boxes (make_tmap_a on the weight).
int gemm_launch_pair(const CUtensorMap& map_a, const CUtensorMap& map_b2, int epi, const GemmArgs& args,
                     cudaStream_t stream, const CUtensorMap* map_b3 = nullptr);
// Swap-AB pair kernel for M <= 256 (gemm_swap.cu): the weight is the MMA's M operand. Returns 1 when the launch is
// not covered (epilogue needs the row-major layout and no split-K applies); the caller then runs gemm_launch_pair /
// gemm_launch. map_w: 128-row boxes over the weight (map_b2). x / ldx: the activation buffer.
int gemm_launch_swap(const CUtensorMap& map_w, const void* x, long long ldx, int epi, const GemmArgs& args,
                     cudaStream_t stream);
bool gemm_swap_enabled();
// Stream-K swap-AB kernel (gemm_sk.cu): every SM pair streams an equal share of the weight's (tile, k-block) work;
// tiles cut between pairs are fixed up in-kernel (no reduce launch). Needs args.sk_ws / sk_flags; returns 1 when the
// launch is not covered.
int gemm_launch_sk(const CUtensorMap& map_w, const void* x, long long ldx, int epi, const GemmArgs& args,
                   cudaStream_t stream);
bool gemm_sk_enabled();          // any epilogue may use it (workspace needed)
bool gemm_sk_enabled(int epi);   // this epilogue uses it
constexpr int SK_FLAG_STRIDE = 32;  // uint32 per flag line
size_t gemm_sk_ws_bytes();          // partial slots for every CTA of a launch
size_t gemm_sk_flag_bytes();
int make_tmap_b64(CUtensorMap* map, const void* B, long long ldb, int N, int K);
int make_tmap_a(CUtensorMap* map, const void* A, long long lda, long long rows, int K);
bool gemm_use_pair(int M);  // pair kernel for M > 128 unless PO_GEMM_1CTA=1
int make_tmap_b(CUtensorMap* map, const void* B, long long ldb, int N, int K);
int num_sms();

// ---- FP8 (E4M3) path: the paper's FP8-weight presets (ps/presets/qwen-32b-fp8.preset, llama-3.3-70b-fp8.preset)
// as W8A8 on tcgen05 kind::f8f6f4. Operands are row-major [rows, K] bytes; K % 128 == 0 (one 128-byte row per
// k-block, the same swizzle and stage geometry as bf16 with BK = 64).
// 128-row (A / pair B half) box map over an E4M3 [rows, K] matrix.
int make_tmap_a_f8(CUtensorMap* map, const void* A, long long lda, long long rows, int K);
// D = dequant(A) . dequant(B)^T with the fused epilogues of gemm_launch_pair (2-CTA pair kernel for every M;
// split-K for short M when args.split_ws is set). args.a_scale / args.b_scale are required.
int gemm_launch_pair_f8(const CUtensorMap& map_a, const CUtensorMap& map_b2, int epi, const GemmArgs& args,
                        cudaStream_t stream);
// Workspace bytes of an FP8 launch of this shape (0 = no split).
size_t gemm_split_ws_bytes_f8(int M, int N, int K);
// Per-row dynamic quantisation: scale[r] = amax(|x[r,:]|) / 448, q[r,c] = e4m3_rn_satfinite(x[r,c] * (448 / amax))
// (scale 0 and q = 0 for an all-zero row). One CTA per row; cols % 16 == 0.
int quantize_rows_e4m3(const __nv_bfloat16* x, long long ldx, int rows, int cols, uint8_t* q, long long ldq,
                       float* scale, cudaStream_t stream);


}  // namespace po
