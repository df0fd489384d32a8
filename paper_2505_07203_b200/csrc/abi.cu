// extern "C" surface of libprefillonly.so (declared in include/prefillonly.h).
#include "../../include/prefillonly.h"
#include "gemm.cuh"
#include <atomic>
#include <cstdio>
#include <string>
#include <cstdarg>

namespace po {
thread_local std::string g_last_error;
int set_error(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

// The op entry points take their scratch from the device's default stream-ordered pool. Keep freed blocks in the
// pool (no release to the driver at every synchronisation), so a per-call workspace costs no driver allocation.
void keep_pool_memory() {
  static std::atomic<uint64_t> done{0};  // one bit per device: each device has its own default pool
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done.fetch_or(bit, std::memory_order_acq_rel);
}
}  // namespace po

extern "C" {

const char* po_last_error(void) { return po::g_last_error.c_str(); }
const char* po_version(void) { return "prefillonly-b200 0.1 (sm_100a)"; }

int po_op_gemm(const void* A, int64_t lda, const void* B, int64_t ldb, void* out, int64_t ldo, float* resid,
               int64_t ldr, int32_t M, int32_t N, int32_t K, int32_t epi, const void* rope_table,
               int32_t pos_offset, int32_t rope_cols, void* stream) {
  if (!A || !B) return po::set_error(PO_ERR_ARG, "po_op_gemm: null operand");
  if (M <= 0 || N % 256 || K % 64 || K <= 0 || N <= 0)
    return po::set_error(PO_ERR_ARG, "po_op_gemm: need M>0, N%%256==0, K%%64==0 (got %d,%d,%d)", M, N, K);
  if (epi == PO_EPI_RESID_F32 ? !resid : !out) return po::set_error(PO_ERR_ARG, "po_op_gemm: null output");
  if (epi == PO_EPI_QKV_ROPE && !rope_table) return po::set_error(PO_ERR_ARG, "po_op_gemm: null rope table");
  po::GemmPlan plan;
  int rc = po::gemm_plan(&plan, A, lda, B, ldb, M, N, K);
  if (rc) return po::set_error(PO_ERR_CUDA, "po_op_gemm: tensor map encode failed (%d)", rc);
  po::GemmArgs args{};
  args.out = out;
  args.ldo = ldo;
  args.resid = resid;
  args.ldr = ldr;
  args.rope = static_cast<const float2*>(rope_table);
  args.pos_offset = pos_offset;
  args.rope_cols = rope_cols;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  po::keep_pool_memory();
  const size_t ws = po::gemm_split_ws_bytes(M, N, K);
  args.split_ws_bytes = ws;
  if (ws && cudaMallocAsync(reinterpret_cast<void**>(&args.split_ws), ws, st) != cudaSuccess)
    return po::set_error(PO_ERR_CUDA, "po_op_gemm: split-K workspace allocation failed");
  // stream-K workspace for short launches (M <= 256): partial slots + flags, zeroed flags, epoch 1
  if (M <= 256 && po::gemm_sk_enabled()) {
    if (cudaMallocAsync(reinterpret_cast<void**>(&args.sk_ws), po::gemm_sk_ws_bytes(), st) != cudaSuccess ||
        cudaMallocAsync(reinterpret_cast<void**>(&args.sk_flags), po::gemm_sk_flag_bytes(), st) != cudaSuccess)
      return po::set_error(PO_ERR_CUDA, "po_op_gemm: stream-K workspace allocation failed");
    cudaMemsetAsync(args.sk_flags, 0, po::gemm_sk_flag_bytes(), st);
    args.sk_epoch = 1;
  }
  rc = po::gemm_run(plan, epi, args, st);
  if (args.split_ws) cudaFreeAsync(args.split_ws, st);
  if (args.sk_ws) cudaFreeAsync(args.sk_ws, st);
  if (args.sk_flags) cudaFreeAsync(args.sk_flags, st);
  if (rc) return po::set_error(PO_ERR_CUDA, "po_op_gemm: launch failed: %s", cudaGetErrorString(cudaGetLastError()));
  return PO_OK;
}

int po_op_gemm_fp8(const void* A, int64_t lda, const float* a_scale, const void* B, int64_t ldb,
                   const float* b_scale, void* out, int64_t ldo, float* resid, int64_t ldr, int32_t M, int32_t N,
                   int32_t K, int32_t epi, const void* rope_table, int32_t pos_offset, int32_t rope_cols,
                   void* stream) {
  if (!A || !B || !a_scale || !b_scale) return po::set_error(PO_ERR_ARG, "po_op_gemm_fp8: null operand or scale");
  if (M <= 0 || N <= 0 || N % 256 || K <= 0 || K % 128)
    return po::set_error(PO_ERR_ARG, "po_op_gemm_fp8: need M>0, N%%256==0, K%%128==0 (got %d,%d,%d)", M, N, K);
  if (epi == PO_EPI_RESID_F32 ? !resid : !out) return po::set_error(PO_ERR_ARG, "po_op_gemm_fp8: null output");
  if (epi == PO_EPI_QKV_ROPE && !rope_table) return po::set_error(PO_ERR_ARG, "po_op_gemm_fp8: null rope table");
  CUtensorMap map_a, map_b;
  if (po::make_tmap_a_f8(&map_a, A, lda, M, K) || po::make_tmap_a_f8(&map_b, B, ldb, N, K))
    return po::set_error(PO_ERR_CUDA, "po_op_gemm_fp8: tensor map encode failed");
  po::GemmArgs args{};
  args.M = M;
  args.N = N;
  args.K = K;
  args.out = out;
  args.ldo = ldo;
  args.resid = resid;
  args.ldr = ldr;
  args.rope = static_cast<const float2*>(rope_table);
  args.pos_offset = pos_offset;
  args.rope_cols = rope_cols;
  args.a_scale = a_scale;
  args.b_scale = b_scale;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  po::keep_pool_memory();
  const size_t ws = po::gemm_split_ws_bytes_f8(M, N, K);
  args.split_ws_bytes = ws;
  if (ws && cudaMallocAsync(reinterpret_cast<void**>(&args.split_ws), ws, st) != cudaSuccess)
    return po::set_error(PO_ERR_CUDA, "po_op_gemm_fp8: split-K workspace allocation failed");
  int rc = po::gemm_launch_pair_f8(map_a, map_b, epi, args, st);
  if (args.split_ws) cudaFreeAsync(args.split_ws, st);
  if (rc) return po::set_error(PO_ERR_CUDA, "po_op_gemm_fp8: launch failed (%d): %s", rc,
                               cudaGetErrorString(cudaGetLastError()));
  return PO_OK;
}

int po_op_quantize_e4m3(const void* x, int64_t ldx, int32_t rows, int32_t cols, void* q, int64_t ldq, float* scale,
                        void* stream) {
  if (!x || !q || !scale) return po::set_error(PO_ERR_ARG, "po_op_quantize_e4m3: null pointer");
  if (rows < 0 || cols <= 0 || cols % 16 || ldx % 8 || ldq % 16 || ldx < cols || ldq < cols)
    return po::set_error(PO_ERR_ARG, "po_op_quantize_e4m3: need cols%%16==0, ldx%%8==0, ldq%%16==0 (got %d,%lld,%lld)",
                         cols, (long long)ldx, (long long)ldq);
  int rc = po::quantize_rows_e4m3(static_cast<const __nv_bfloat16*>(x), ldx, rows, cols, static_cast<uint8_t*>(q), ldq,
                                  scale, static_cast<cudaStream_t>(stream));
  if (rc) return po::set_error(PO_ERR_CUDA, "po_op_quantize_e4m3: launch failed (%d)", rc);
  return PO_OK;
}

}  // extern "C"
