/* prefillonly.h — C-ABI of the B200-native PrefillOnly engine (libprefillonly.so).
 *
 * The reference (arxiv 2505.07203, /root/reference/pkg) is a pure-Python simulator with no FFI.
 * Each entry point below names the reference interface it replaces; the Python host package
 * (paper_2505_07203_b200/) binds these with ctypes, exactly as a reference maintainer would (see
 * INTEGRATION.md).
 *
 * Conventions
 *   - Every function returns 0 on success or a negative PO_ERR_* status; po_last_error() gives text.
 *   - Device pointers are raw CUDA device addresses (e.g. torch.Tensor.data_ptr()); host pointers are
 *     plain CPU memory owned by the caller, which may be reused as soon as the call returns.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).
 *   - No torch types cross this boundary.
 */
#ifndef PREFILLONLY_H
#define PREFILLONLY_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes, mapped onto the reference error taxonomy. */
#define PO_OK 0
#define PO_ERR_CONFIG (-2)   /* GeometryError / NumericsError / CostError  (ps/geometry.py:18, ps/numerics.py:26) */
#define PO_ERR_CAPACITY (-3) /* CapacityError: request beyond MIL             (ps/costs.py:40-45,270-274)        */
#define PO_ERR_CUDA (-4)     /* CUDA runtime / launch failure                                                    */
#define PO_ERR_ARG (-5)      /* invalid argument (null pointer, bad shape)                                       */
#define PO_ERR_POOL (-6)     /* prefix-pool slot out of range, or one slot named twice in a request              */

const char* po_last_error(void);
const char* po_version(void);

/* ------------------------------------------------------------------------------------------------
 * Kernel-level operators (device pointers). These are the building blocks of po_prefill and are
 * exported so parity tests can check each kernel against the CPU oracle in isolation.
 * ------------------------------------------------------------------------------------------------ */

/* Epilogue selectors for po_op_gemm. */
#define PO_EPI_BF16 0      /* out(bf16)[m,n] = acc                                                        */
#define PO_EPI_RESID_F32 1 /* resid(f32)[m,n] += acc      (in-place residual)           */
#define PO_EPI_SILU_MUL 2  /* out(bf16)[m,n/2] = silu(gate)*up, gate/up interleaved by 16 columns        */
#define PO_EPI_QKV_ROPE 3  /* out(bf16)[m,n] = acc with rotate-half RoPE on columns < rope_cols         */
#define PO_EPI_F32 4       /* out(f32)[m,n] = acc                                                        */

/* D = A[M,K] . B[N,K]^T on tcgen05 tensor cores (bf16 in, fp32 accumulate).
 * Replaces the chunked np.matmul stages of block_forward_hybrid (ps/numerics.py:236-239,244-255,259-274).
 * Requires N % 256 == 0 and K % 64 == 0; lda/ldb/ldo/ldr in elements. */
int po_op_gemm(const void* A, int64_t lda, const void* B, int64_t ldb, void* out, int64_t ldo, float* resid,
               int64_t ldr, int32_t M, int32_t N, int32_t K, int32_t epi, const void* rope_table,
               int32_t pos_offset, int32_t rope_cols, void* stream);

/* FP8 (W8A8 E4M3) variant of po_op_gemm for the paper's FP8-weight presets (ps/presets/qwen-32b-fp8.preset:1-16,
 * ps/presets/llama-3.3-70b-fp8.preset:1-15; tcgen05 kind::f8f6f4). A [M,K] and B [N,K] are E4M3 bytes (lda/ldb
 * in bytes), a_scale [M] / b_scale [N] fp32 dequantisation scales: acc[m,n] * a_scale[m] * b_scale[n] feeds the
 * same epilogues as po_op_gemm. Requires N % 256 == 0 and K % 128 == 0. */
int po_op_gemm_fp8(const void* A, int64_t lda, const float* a_scale, const void* B, int64_t ldb,
                   const float* b_scale, void* out, int64_t ldo, float* resid, int64_t ldr, int32_t M, int32_t N,
                   int32_t K, int32_t epi, const void* rope_table, int32_t pos_offset, int32_t rope_cols,
                   void* stream);

/* A chain of one or two GEMMs through the persistent weight-streaming kernel that runs prefix hits' layer GEMMs
 * (M <= 256 rows; stream-K split of the weight matrix over the SM pairs, in-kernel fix-up, grid barrier between the
 * phases): out1(bf16)[M,N1] = A[M,K] . B1[N1,K]^T, then, when B2 is not null, out2(bf16)[M,N2] = out1 . B2[N2,N1]^T
 * in the same launch. Replaces the chunked np.matmul stages (ps/numerics.py:244-255) for short miss suffixes.
 * Requires 1 <= M <= 256, N % 256 == 0, K % 64 == 0 (N1 % 64 == 0 for the second phase). */
int po_op_stream_gemm(const void* A, int64_t lda, const void* B1, int64_t ldb1, void* out1, int64_t ldo1, int32_t M,
                      int32_t N1, int32_t K, const void* B2, int64_t ldb2, void* out2, int64_t ldo2, int32_t N2,
                      void* stream);

/* Per-row dynamic E4M3 quantisation of a bf16 [rows, cols] matrix (activations before an FP8 GEMM, or weight
 * rows = output channels): scale[r] = amax_r / 448, q[r,c] = e4m3_satfinite_rn(x[r,c] * (448 / amax_r)).
 * cols % 16 == 0, ldx % 8 == 0, ldq % 16 == 0 (elements / bytes). */
int po_op_quantize_e4m3(const void* x, int64_t ldx, int32_t rows, int32_t cols, void* q, int64_t ldq, float* scale,
                        void* stream);

/* Causal GQA attention over one layer's qkv buffer (bf16 [n_total, ld]: Q | K | V columns, head_dim 128).
 * Rows [0, q_offset) are cached-prefix rows that act only as keys; the output ctx (bf16 [n_total-q_offset,
 * ldo]) holds the n_total-q_offset query rows. Replaces _attention (ps/numerics.py:132-146) generalised to
 * GQA with prefix hits ((n^2 - n_c^2)/2 pairs, ps/costs.py:275-277). n_heads/n_kv_heads must be even. */
int po_op_attention(const void* qkv, int64_t ld, int32_t n_total, int32_t q_offset, int32_t n_heads,
                    int32_t n_kv_heads, void* out, int64_t ldo, void* stream);

/* ------------------------------------------------------------------------------------------------
 * Engine (one per GPU; one request in flight, ps/sim.py:4-9). Replaces the engine slot
 * execute_time(variant, geom, gpu, params, n_input, n_cached) called from sim.run.start_next
 * (ps/costs.py:259-280, ps/sim.py:217-220): instead of returning modelled seconds, po_prefill runs the
 * hybrid-prefill forward and the allowed-row LM head and reports measured device time.
 * ------------------------------------------------------------------------------------------------ */
typedef struct po_model_cfg {
  int32_t num_layers;        /* ModelGeometry.num_layers            (ps/geometry.py:29-33)              */
  int32_t hidden;            /* ModelGeometry.hidden_size                                               */
  int32_t n_heads;           /* query heads (absent in reference; Llama config)                        */
  int32_t n_kv_heads;        /* ModelGeometry.num_kv_heads                                              */
  int32_t head_dim;          /* ModelGeometry.head_dim (must be 128)                                    */
  int32_t intermediate;      /* ModelGeometry.intermediate_size                                         */
  int32_t vocab;             /* vocabulary rows of embed / lm_head                                      */
  float rms_eps;             /* RMSNorm epsilon                                                         */
  float rope_theta;          /* RoPE base                                                               */
  int32_t rope_scaling;      /* 0 = none, 1 = llama3                                                    */
  float rope_factor, rope_low_freq_factor, rope_high_freq_factor;
  int32_t rope_original_max_pos;
  int32_t max_tokens;        /* largest request the arena serves (the MIL, ps/geometry.py:203-212)     */
  int32_t chunk;             /* hybrid-prefill MLP chunk rows (DEFAULT_CHUNK = 8192, ps/geometry.py:14) */
  int32_t block_tokens;      /* prefix-pool block (CacheConfig.block_tokens = 16, ps/cache.py:65-80)   */
  int64_t pool_blocks;       /* prefix-pool capacity in blocks; < 0 = size by a profile run            */
  double pool_mem_fraction;  /* profile run: fraction of HBM left after the arena given to the pool    */
  int32_t last_row_only;     /* 1: in the last layer run attention/O/MLP for the final row only (exact:    */
                             /*    only that row reaches the LM head); 0: every row through every layer  */
  int32_t qkv_bias;          /* 1: q/k/v projections carry a bias (Qwen2), added before RoPE               */
  int32_t weight_fp8;        /* 1: layer weights stored E4M3 with per-output-channel scales (the FP8 presets,   */
                             /*    ps/presets/qwen-32b-fp8.preset:1-16); GEMMs run W8A8 (kind::f8f6f4) with   */
                             /*    per-row dynamic activation scales. Embedding and LM head stay bf16.       */
} po_model_cfg;

typedef struct po_engine po_engine;

/* Allocate weights (counter-hash random init from `seed`, bit-reproducible by oracle/), the activation
 * arena for cfg->max_tokens, the one-layer K/V buffer and the prefix pool. */
int po_init(int32_t device, const po_model_cfg* cfg, uint64_t seed, po_engine** out);
int po_free(po_engine* e);

/* One prefill-only request: tokens[n] (uint32 ids, embedded as id % vocab), n_cached prefix tokens already
 * resident in the pool (multiple of block_tokens). pool_block_ids[b] for b < n_blocks: for cached blocks
 * (b < n_cached/block_tokens) the slot holding block b; for later blocks the slot to admit block b into, or
 * -1 (suffix discard, ps/cache.py:143-159). Outputs (host): logits/probs over the allowed ids (softmax
 * restricted to them) and the argmax index into `allowed` (first maximum). PO_ERR_CAPACITY when
 * n > max_tokens (CapacityError, ps/costs.py:270-274); PO_ERR_POOL when a slot is out of range or named twice in
 * one request (an admitted block may not reuse a slot this request reads or admits elsewhere). */
int po_prefill(po_engine* e, const uint32_t* tokens, int32_t n, int32_t n_cached, const int32_t* allowed,
               int32_t n_allowed, const int32_t* pool_block_ids, int32_t n_blocks, float* out_logits,
               float* out_probs, int32_t* out_argmax, void* stream);

/* po_prefill split in two, so a serving loop can take its next scheduling decision while this forward runs
 * (ps/sim.py:217-229 decides at completion; serving.Server's lookahead decides one request ahead).
 * po_prefill_submit validates and stages the request (host buffers are copied; the caller may reuse them on
 * return), enqueues the forward on `stream` and returns a ticket. po_prefill_query sets *done when the ticket's
 * forward and output copies have completed; po_prefill_wait blocks until then and copies the outputs
 * (service_ms: device time of the forward incl. its H2D/D2H copies; may be NULL). Staging rotates over 4 entries:
 * at most 3 tickets may be outstanding, a ticket's outputs are lost once 4 newer submits have recycled its entry
 * (wait/query then return PO_ERR_ARG). po_prefill == submit + wait. */
int po_prefill_submit(po_engine* e, const uint32_t* tokens, int32_t n, int32_t n_cached, const int32_t* allowed,
                      int32_t n_allowed, const int32_t* pool_block_ids, int32_t n_blocks, int64_t* ticket,
                      void* stream);
int po_prefill_query(po_engine* e, int64_t ticket, int32_t* done);
int po_prefill_wait(po_engine* e, int64_t ticket, float* out_logits, float* out_probs, int32_t* out_argmax,
                    float* service_ms);

/* Same forward on device-resident inputs (d_tokens: all n uint32 ids; d_allowed: n_allowed ids) with device
 * outputs; asynchronous on `stream` (NULL = the engine's stream, see po_engine_stream). pool_block_ids is a
 * host array as in po_prefill. Used to time the hot path with inputs already in HBM. */
int po_prefill_device(po_engine* e, const uint32_t* d_tokens, int32_t n, int32_t n_cached, const int32_t* d_allowed,
                      int32_t n_allowed, const int32_t* pool_block_ids, int32_t n_blocks, float* d_logits,
                      float* d_probs, int32_t* d_argmax, void* stream);
int po_engine_stream(po_engine* e, void** stream);
/* Kernel launches issued by the last forward. */
int po_last_launches(po_engine* e, int32_t* n);
/* Per-kernel-class CUDA-event timing over the forwards issued between begin and end. Classes: 0 embed,
 * 1 rmsnorm, 2 kv_gather, 3 gemm_qkv_rope, 4 kv_scatter, 5 attention, 6 gemm_o_resid, 7 gemm_gate_up_silu,
 * 8 gemm_down_resid, 9 lm_head. */
int po_profile_begin(po_engine* e);
int po_profile_end(po_engine* e, float* ms_per_class, int32_t* launches_per_class, int32_t n_classes);

/* Device milliseconds of the last po_prefill (CUDA events around the forward on the engine stream). */
int po_last_service_ms(po_engine* e, float* ms);

/* Drop pool slots (metadata-only: slots are overwritten on reuse; validates the ids). */
int po_pool_evict(po_engine* e, const int32_t* slots, int32_t n);

/* Engine facts: [0] pool_blocks, [1] weight bytes, [2] arena bytes, [3] pool bytes, [4] bytes per pool block,
 * [5] max_tokens, [6] device free bytes after init, [7] split-KV / split-K workspace bytes. */
int po_engine_info(po_engine* e, int64_t* out, int32_t n);

/* Overwrite one weight tensor from host memory (logical, un-interleaved layout; bf16 except norms = fp32).
 * kind: 0 embed, 1 attn_norm, 2 wq, 3 wk, 4 wv, 5 wo, 6 mlp_norm, 7 w_gate, 8 w_up, 9 w_down, 10 final_norm,
 * 11 lm_head, 12 qkv bias (fp32, [(Hq+2Hkv)*128]). */
int po_load_weight(po_engine* e, int32_t kind, int32_t layer, const void* host, int64_t nelem);

#ifdef __cplusplus
}
#endif
#endif /* PREFILLONLY_H */
