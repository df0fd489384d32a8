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
#define PO_ERR_POOL (-6)     /* prefix-pool slot out of range                                                    */

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

/* Causal GQA attention over one layer's qkv buffer (bf16 [n_total, ld]: Q | K | V columns, head_dim 128).
 * Rows [0, q_offset) are cached-prefix rows that act only as keys; the output ctx (bf16 [n_total-q_offset,
 * ldo]) holds the n_total-q_offset query rows. Replaces _attention (ps/numerics.py:132-146) generalised to
 * GQA with prefix hits ((n^2 - n_c^2)/2 pairs, ps/costs.py:275-277). n_heads/n_kv_heads must be even. */
int po_op_attention(const void* qkv, int64_t ld, int32_t n_total, int32_t q_offset, int32_t n_heads,
                    int32_t n_kv_heads, void* out, int64_t ldo, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PREFILLONLY_H */
