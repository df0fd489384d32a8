// PrefillOnly engine: weights, activation arena, one-layer K/V buffer, prefix pool, hybrid-prefill forward.
//
// Forward of one request (n tokens, n_c cached, ps/numerics.py:215-275 generalised to Llama):
//   resid = embed(tokens[n_c:])                                            fp32 [n_miss, h]
//   for each layer:                                     (KV of this layer only: qkv is reused across layers)
//     xn   = rmsnorm(resid) * g_attn                                       bf16 [n_miss, h]
//     qkv[:n_c, kv]   = gather(prefix pool, cached blocks)                 bf16 K/V of the cached prefix
//     qkv[n_c:]       = xn . Wqkv^T  (+RoPE epilogue)                      tcgen05 GEMM
//     pool[admitted]  = K/V of the admitted rows (stored by the QKV epilogue) prefix-pool admission
//     ctx  = causal GQA attention(qkv, q_offset = n_c)                     full length, tcgen05 FA
//     resid += ctx . Wo^T                                                  residual epilogue, in place
//     for chunk of rows:                                                   hybrid: MLP chunked
//       xn[chunk]    = rmsnorm(resid[chunk]) * g_mlp
//       act          = silu(xn Wg^T) * (xn Wu^T)                           one GEMM, SiLU.mul epilogue
//       resid[chunk] += act . Wd^T                                         residual epilogue, in place
//   logits over allowed ids = lm_head[allowed] . rmsnorm(resid[last]) * g_final
#include "../../include/prefillonly.h"
#include "gemm.cuh"
#include "kernels.cuh"
#include "attention.cuh"
#include "stream.cuh"
#include "mlp.cuh"
#include <cmath>
#include <cstring>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <algorithm>
#include <vector>

namespace po {
int set_error(int code, const char* fmt, ...);
}  // namespace po

struct po_engine {
  po_model_cfg cfg;
  int device = 0;
  uint64_t seed = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // weights
  __nv_bfloat16* embed = nullptr;
  __nv_bfloat16* lm_head = nullptr;
  float* final_norm = nullptr;
  struct Layer {
    __nv_bfloat16 *wqkv, *wo, *wgu, *wdown;
    float *attn_norm, *mlp_norm;
    float* bqkv = nullptr;  // q/k/v bias (qkv_bias models), fp32 holding bf16 values
    CUtensorMap map_qkv, map_o, map_gu, map_down;      // 256-row boxes (1-CTA kernel)
    CUtensorMap map2_qkv, map2_o, map2_gu, map2_down;  // 128-row boxes (2-CTA pair kernel)
    CUtensorMap map3_qkv, map3_o, map3_gu, map3_down;  // 64-row boxes (narrow pair tiles, small M)
    // weight_fp8: E4M3 copies [rows, K] with fp32 per-row (output-channel) scales replace the bf16 matrices
    uint8_t *q_qkv = nullptr, *q_o = nullptr, *q_gu = nullptr, *q_down = nullptr;
    float *s_qkv = nullptr, *s_o = nullptr, *s_gu = nullptr, *s_down = nullptr;
    CUtensorMap f8_qkv, f8_o, f8_gu, f8_down;  // 128-row boxes of 128 bytes (pair kernel)
  };
  std::vector<Layer> layers;
  // arena
  float* resid = nullptr;
  __nv_bfloat16* xn = nullptr;  // attention output (ctx)
  __nv_bfloat16* xg = nullptr;  // bf16(resid . gamma): the folded-RMSNorm GEMM input (see GemmArgs)
  float* ss_attn = nullptr;     // per-row, per-128-column sums of resid^2 feeding the next attention norm
  float* ss_mlp = nullptr;      // ... feeding the next MLP norm
  __nv_bfloat16* qkv = nullptr;
  __nv_bfloat16* act = nullptr;
  float2* rope = nullptr;
  float* gemm_ws = nullptr;  // split-K partials for small-M (prefix-hit) GEMMs
  size_t gemm_ws_bytes = 0;
  void* attn_ws = nullptr;  // split-KV partials for short-query (prefix-hit) requests
  size_t attn_ws_bytes = 0;
  CUtensorMap map_xn, map_ctx, map_act, map_xg;
  // weight_fp8: per-row E4M3 copies of the GEMM inputs (xg, ctx, act) and their dequantisation scales
  uint8_t *xg8 = nullptr, *ctx8 = nullptr, *act8 = nullptr;
  float *xg_s = nullptr, *ctx_s = nullptr, *act_s = nullptr;
  CUtensorMap map_xg8, map_ctx8, map_act8;
  // per-request device staging
  uint32_t* d_tokens = nullptr;
  int* d_slots = nullptr;   // the current request's ring entry (below)
  int* d_kvslot = nullptr;  // per 16-token block: admission slot in the prefix pool, or -1
  // Block tables go through a ring of STAGE_RING pinned/device buffer pairs: po_prefill_device returns before its
  // forward (and the H2D copy of its tables) ran, so the next call must not overwrite those pinned buffers. Each
  // entry is reused only after the event recorded behind the forward that used it has completed.
  static constexpr int STAGE_RING = 4;
  int* ring_h_slots[STAGE_RING] = {};
  int* ring_h_kvslot[STAGE_RING] = {};
  int* ring_d_slots[STAGE_RING] = {};
  int* ring_d_kvslot[STAGE_RING] = {};
  cudaEvent_t ring_ev[STAGE_RING] = {};
  // per entry: the request's pinned token / allowed-id staging, its pinned outputs, device-time events and the
  // ticket of the po_prefill_submit that owns it (po_prefill_wait reads the outputs back through the ticket)
  uint32_t* ring_h_tokens[STAGE_RING] = {};
  int* ring_h_allowed[STAGE_RING] = {};
  float* ring_h_logits[STAGE_RING] = {};
  float* ring_h_probs[STAGE_RING] = {};
  int* ring_h_argmax[STAGE_RING] = {};
  cudaEvent_t ring_ev0[STAGE_RING] = {}, ring_ev1[STAGE_RING] = {};
  int64_t ring_ticket[STAGE_RING] = {};
  int ring_n_allowed[STAGE_RING] = {};
  int ring_next = 0;
  int cur_ring = 0;  // entry of the request being staged
  int64_t next_ticket = 0;
  int* d_allowed = nullptr;
  float* d_logits = nullptr;
  float* d_probs = nullptr;
  int* d_argmax = nullptr;
  // pinned host staging
  uint32_t* h_tokens = nullptr;
  int* h_slots = nullptr;
  int* h_kvslot = nullptr;
  int* h_allowed = nullptr;
  float* h_logits = nullptr;
  float* h_probs = nullptr;
  int* h_argmax = nullptr;
  // prefix pool [slot][layer][block_tokens][kv_dim]
  __nv_bfloat16* pool = nullptr;
  int64_t pool_blocks = 0;
  int64_t weight_bytes = 0, arena_bytes = 0, pool_bytes = 0, free_after = 0, workspace_bytes = 0;
  std::vector<void*> allocs;
  unsigned int* lm_ticket = nullptr;      // multi-CTA LM head: CTAs finished (the last one runs the softmax)
  int* mlp_cnt = nullptr;                 // fused MLP launch: per-piece completion counters + exit ticket
  unsigned int* mlp_ticket = nullptr;
  int* mlp_next = nullptr;
  int mlp_piece_max = 0;                  // rows per piece of the act ring (two pieces = chunk rows)
  std::vector<int> piece_plan;            // MLP piece rows of the last planned row count (plan_mlp_pieces)
  int piece_plan_rows = -1;
  float* sk_ws = nullptr;       // stream-K short-launch GEMMs: per-CTA partial slots and flags (gemm_sk.cu)
  uint32_t* sk_flags = nullptr;
  uint32_t sk_epoch = 0;
  // persistent weight-streaming kernel (prefix hits): partial tiles, fix-up flags, grid-barrier counter
  float* stream_ws = nullptr;
  size_t stream_ws_bytes = 0;
  uint32_t* stream_flags = nullptr;
  size_t stream_n_flags = 0;
  unsigned long long* stream_bar = nullptr;
  unsigned long long stream_bar_base = 0;
  uint32_t stream_tag = 1;
  bool act_persist = false;  // the MLP chunk buffer is pinned in L2 (persisting access-policy window)
  std::vector<uint32_t> slot_stamp;  // per pool slot: the last request that named it (collision check)
  uint32_t stamp_gen = 0;
  float last_ms = 0.f;
  float last_enqueue_ms = 0.f;  // host time to enqueue the forward (launch-bound when it approaches last_ms)
  int last_launches = 0;
  // per-kernel-class CUDA-event timing (bench roofline)
  bool profiling = false;
  int prof_used = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_events;
  std::vector<int> prof_class;

  int qkv_cols() const { return (cfg.n_heads + 2 * cfg.n_kv_heads) * cfg.head_dim; }
  int kv_dim() const { return 2 * cfg.n_kv_heads * cfg.head_dim; }
  int ctx_cols() const { return cfg.n_heads * cfg.head_dim; }
  int64_t block_bytes() const { return (int64_t)cfg.num_layers * cfg.block_tokens * kv_dim() * 2; }
  bool fp8() const { return cfg.weight_fp8 != 0; }
};

namespace {
using po::set_error;

// tensor ids of the counter-hash init (oracle/llama_ref.py mirrors these)
constexpr uint32_t TID_EMBED = 0xFFFF0, TID_FINAL_NORM = 0xFFFF1, TID_LM_HEAD = 0xFFFF2;
enum { K_ATTN_NORM = 0, K_Q = 1, K_K = 2, K_V = 3, K_O = 4, K_MLP_NORM = 5, K_GATE = 6, K_UP = 7, K_DOWN = 8,
       K_QKV_BIAS = 9 };
inline uint32_t layer_tid(int layer, int kind) { return static_cast<uint32_t>(layer) * 16u + kind; }
inline float fan_scale(int fan_in) { return static_cast<float>(1.0 / std::sqrt(static_cast<double>(fan_in))); }

template <typename T>
int dalloc(po_engine* e, T** p, size_t bytes, int64_t* counter) {
  void* q = nullptr;
  if (cudaMalloc(&q, bytes ? bytes : 16) != cudaSuccess) return -1;
  e->allocs.push_back(q);
  *p = static_cast<T*>(q);
  if (counter) *counter += bytes;
  return 0;
}
template <typename T>
int halloc(T** p, size_t bytes) {
  return cudaMallocHost(reinterpret_cast<void**>(p), bytes ? bytes : 16) == cudaSuccess ? 0 : -1;
}

// Llama-3 RoPE inverse frequencies in double, rounded once to fp32 (oracle/llama_ref.py: rope_inv_freq)
std::vector<float> rope_inv_freq(const po_model_cfg& c) {
  std::vector<float> out(c.head_dim / 2);
  for (int i = 0; i < c.head_dim / 2; ++i) {
    double f = 1.0 / std::pow(static_cast<double>(c.rope_theta), (2.0 * i) / c.head_dim);
    if (c.rope_scaling == 1) {
      const double orig = c.rope_original_max_pos;
      const double low_wl = orig / c.rope_low_freq_factor, high_wl = orig / c.rope_high_freq_factor;
      const double wl = 2.0 * M_PI / f;
      if (wl > low_wl) {
        f = f / c.rope_factor;
      } else if (wl >= high_wl) {
        const double s = (orig / wl - c.rope_low_freq_factor) / (c.rope_high_freq_factor - c.rope_low_freq_factor);
        f = (1.0 - s) * f / c.rope_factor + s * f;
      }
    }
    out[i] = static_cast<float>(f);
  }
  return out;
}

int validate_cfg(const po_model_cfg& c) {
  if (c.num_layers <= 0 || c.hidden <= 0 || c.n_heads <= 0 || c.n_kv_heads <= 0 || c.intermediate <= 0 ||
      c.vocab <= 0 || c.max_tokens <= 0 || c.chunk <= 0 || c.block_tokens <= 0)
    return set_error(PO_ERR_CONFIG, "po_init: all shape counts must be positive");
  if (c.head_dim != 128) return set_error(PO_ERR_CONFIG, "po_init: head_dim must be 128 (got %d)", c.head_dim);
  if (c.n_heads % c.n_kv_heads)
    return set_error(PO_ERR_CONFIG, "po_init: n_heads must be a multiple of n_kv_heads");
  if (c.hidden % 256 || c.intermediate % 128 || ((c.n_heads + 2 * c.n_kv_heads) * 128) % 256)
    return set_error(PO_ERR_CONFIG, "po_init: hidden %% 256, intermediate %% 128 and qkv width %% 256 required");
  if (c.hidden > 8192) return set_error(PO_ERR_CONFIG, "po_init: hidden > 8192 unsupported by the LM-head kernel");
  // the QKV-epilogue admission (pool_row), pool-direct attention and the pool layout use 16-token blocks
  if (c.block_tokens != 16)
    return set_error(PO_ERR_CONFIG, "po_init: block_tokens must be 16 (got %d)", c.block_tokens);
  return 0;
}
}  // namespace

extern "C" {

int po_free(po_engine* e) {
  if (!e) return PO_OK;
  cudaSetDevice(e->device);
  if (e->stream) cudaStreamSynchronize(e->stream);
  if (e->act_persist) {  // hand the persisting L2 carve-out back
    cudaCtxResetPersistingL2Cache();
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
  }
  for (void* p : e->allocs) cudaFree(p);
  for (int i = 0; i < po_engine::STAGE_RING; ++i) {
    cudaFreeHost(e->ring_h_slots[i]);
    cudaFreeHost(e->ring_h_kvslot[i]);
    cudaFreeHost(e->ring_h_tokens[i]);
    cudaFreeHost(e->ring_h_allowed[i]);
    cudaFreeHost(e->ring_h_logits[i]);
    cudaFreeHost(e->ring_h_probs[i]);
    cudaFreeHost(e->ring_h_argmax[i]);
    if (e->ring_ev[i]) cudaEventDestroy(e->ring_ev[i]);
    if (e->ring_ev0[i]) cudaEventDestroy(e->ring_ev0[i]);
    if (e->ring_ev1[i]) cudaEventDestroy(e->ring_ev1[i]);
  }
  for (auto& pr : e->prof_events) {
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  if (e->ev0) cudaEventDestroy(e->ev0);
  if (e->ev1) cudaEventDestroy(e->ev1);
  if (e->stream) cudaStreamDestroy(e->stream);
  delete e;
  return PO_OK;
}

int po_init(int32_t device, const po_model_cfg* cfg, uint64_t seed, po_engine** out) {
  if (!cfg || !out) return set_error(PO_ERR_ARG, "po_init: null argument");
  *out = nullptr;
  if (int rc = validate_cfg(*cfg)) return rc;
  if (cudaSetDevice(device) != cudaSuccess) return set_error(PO_ERR_CUDA, "po_init: cudaSetDevice(%d) failed", device);
  po_engine* e = new po_engine();
  e->cfg = *cfg;
  e->device = device;
  e->seed = seed;
  const po_model_cfg& c = e->cfg;
  auto fail = [&](int code, const char* what) {
    int rc = set_error(code, "po_init: %s (%s)", what, cudaGetErrorString(cudaGetLastError()));
    po_free(e);
    return rc;
  };
  if (cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&e->ev0) != cudaSuccess || cudaEventCreate(&e->ev1) != cudaSuccess)
    return fail(PO_ERR_CUDA, "stream/event creation failed");
  const int h = c.hidden, I = c.intermediate, L = c.num_layers;
  const int qkvc = e->qkv_cols(), ctxc = e->ctx_cols();
  const long long T = c.max_tokens;
  cudaStream_t s = e->stream;

  // ---- weights (counter-hash init; bf16, norms as fp32 holding bf16 values)
  if (dalloc(e, &e->embed, (size_t)c.vocab * h * 2, &e->weight_bytes) ||
      dalloc(e, &e->lm_head, (size_t)c.vocab * h * 2, &e->weight_bytes) ||
      dalloc(e, &e->final_norm, (size_t)h * 4, &e->weight_bytes))
    return fail(PO_ERR_CUDA, "weight allocation failed");
  po::launch_init_bf16(e->embed, c.vocab, h, seed, TID_EMBED, 0, 1.0f, po::INIT_PLAIN, s);
  po::launch_init_bf16(e->lm_head, c.vocab, h, seed, TID_LM_HEAD, 0, fan_scale(h), po::INIT_PLAIN, s);
  po::launch_init_norm(e->final_norm, h, seed, TID_FINAL_NORM, s);
  e->layers.resize(L);
  // weight_fp8: each bf16 matrix is generated into a scratch buffer (not counted as weights) and quantised per output
  // row into its E4M3 copy, so the random init is the bf16 model's, rounded once more
  const bool f8 = e->fp8();
  __nv_bfloat16* wtmp = nullptr;
  if (f8) {
    const size_t most = std::max(std::max((size_t)qkvc * h, (size_t)h * ctxc), std::max((size_t)2 * I * h, (size_t)h * I));
    if (cudaMalloc(&wtmp, most * 2) != cudaSuccess) return fail(PO_ERR_CUDA, "weight scratch allocation failed");
  }
  auto quant = [&](int rows, int cols, uint8_t* q, float* sc) {
    return po::quantize_rows_e4m3(wtmp, cols, rows, cols, q, cols, sc, s);
  };
  int wrc = 0;
  for (int l = 0; l < L && !wrc; ++l) {
    auto& ly = e->layers[l];
    if (!f8 && (dalloc(e, &ly.wqkv, (size_t)qkvc * h * 2, &e->weight_bytes) ||
                dalloc(e, &ly.wo, (size_t)h * ctxc * 2, &e->weight_bytes) ||
                dalloc(e, &ly.wgu, (size_t)2 * I * h * 2, &e->weight_bytes) ||
                dalloc(e, &ly.wdown, (size_t)h * I * 2, &e->weight_bytes)))
      wrc = -1;
    if (f8 && (dalloc(e, &ly.q_qkv, (size_t)qkvc * h, &e->weight_bytes) ||
               dalloc(e, &ly.s_qkv, (size_t)qkvc * 4, &e->weight_bytes) ||
               dalloc(e, &ly.q_o, (size_t)h * ctxc, &e->weight_bytes) ||
               dalloc(e, &ly.s_o, (size_t)h * 4, &e->weight_bytes) ||
               dalloc(e, &ly.q_gu, (size_t)2 * I * h, &e->weight_bytes) ||
               dalloc(e, &ly.s_gu, (size_t)2 * I * 4, &e->weight_bytes) ||
               dalloc(e, &ly.q_down, (size_t)h * I, &e->weight_bytes) ||
               dalloc(e, &ly.s_down, (size_t)h * 4, &e->weight_bytes)))
      wrc = -1;
    if (wrc || dalloc(e, &ly.attn_norm, (size_t)h * 4, &e->weight_bytes) ||
        dalloc(e, &ly.mlp_norm, (size_t)h * 4, &e->weight_bytes)) {
      cudaFree(wtmp);
      return fail(PO_ERR_CUDA, "weight allocation failed");
    }
    const int qrows = c.n_heads * c.head_dim, kvrows = c.n_kv_heads * c.head_dim;
    __nv_bfloat16* wqkv = f8 ? wtmp : ly.wqkv;
    po::launch_init_bf16(wqkv, qrows, h, seed, layer_tid(l, K_Q), 0, fan_scale(h), po::INIT_PLAIN, s);
    po::launch_init_bf16(wqkv + (size_t)qrows * h, kvrows, h, seed, layer_tid(l, K_K), 0, fan_scale(h),
                         po::INIT_PLAIN, s);
    po::launch_init_bf16(wqkv + (size_t)(qrows + kvrows) * h, kvrows, h, seed, layer_tid(l, K_V), 0, fan_scale(h),
                         po::INIT_PLAIN, s);
    if (f8) wrc |= quant(qkvc, h, ly.q_qkv, ly.s_qkv);
    po::launch_init_bf16(f8 ? wtmp : ly.wo, h, ctxc, seed, layer_tid(l, K_O), 0, fan_scale(ctxc), po::INIT_PLAIN, s);
    if (f8) wrc |= quant(h, ctxc, ly.q_o, ly.s_o);
    po::launch_init_bf16(f8 ? wtmp : ly.wgu, 2 * I, h, seed, layer_tid(l, K_GATE), layer_tid(l, K_UP), fan_scale(h),
                         po::INIT_GATE_UP, s);
    if (f8) wrc |= quant(2 * I, h, ly.q_gu, ly.s_gu);
    po::launch_init_bf16(f8 ? wtmp : ly.wdown, h, I, seed, layer_tid(l, K_DOWN), 0, fan_scale(I), po::INIT_PLAIN, s);
    if (f8) wrc |= quant(h, I, ly.q_down, ly.s_down);
    po::launch_init_norm(ly.attn_norm, h, seed, layer_tid(l, K_ATTN_NORM), s);
    if (c.qkv_bias) {
      if (dalloc(e, &ly.bqkv, (size_t)qkvc * 4, &e->weight_bytes)) {
        cudaFree(wtmp);
        return fail(PO_ERR_CUDA, "bias allocation failed");
      }
      po::launch_init_bias(ly.bqkv, qkvc, seed, layer_tid(l, K_QKV_BIAS), s);
    }
    po::launch_init_norm(ly.mlp_norm, h, seed, layer_tid(l, K_MLP_NORM), s);
    if (f8) {
      if (po::make_tmap_a_f8(&ly.f8_qkv, ly.q_qkv, h, qkvc, h) || po::make_tmap_a_f8(&ly.f8_o, ly.q_o, ctxc, h, ctxc) ||
          po::make_tmap_a_f8(&ly.f8_gu, ly.q_gu, h, 2 * I, h) || po::make_tmap_a_f8(&ly.f8_down, ly.q_down, I, h, I))
        wrc = -2;
    } else if (po::make_tmap_b(&ly.map_qkv, ly.wqkv, h, qkvc, h) || po::make_tmap_b(&ly.map_o, ly.wo, ctxc, h, ctxc) ||
               po::make_tmap_b(&ly.map_gu, ly.wgu, h, 2 * I, h) || po::make_tmap_b(&ly.map_down, ly.wdown, I, h, I) ||
               po::make_tmap_a(&ly.map2_qkv, ly.wqkv, h, qkvc, h) || po::make_tmap_a(&ly.map2_o, ly.wo, ctxc, h, ctxc) ||
               po::make_tmap_a(&ly.map2_gu, ly.wgu, h, 2 * I, h) || po::make_tmap_a(&ly.map2_down, ly.wdown, I, h, I) ||
               po::make_tmap_b64(&ly.map3_qkv, ly.wqkv, h, qkvc, h) ||
               po::make_tmap_b64(&ly.map3_o, ly.wo, ctxc, h, ctxc) ||
               po::make_tmap_b64(&ly.map3_gu, ly.wgu, h, 2 * I, h) ||
               po::make_tmap_b64(&ly.map3_down, ly.wdown, I, h, I)) {
      wrc = -2;
    }
  }
  if (wtmp) {
    cudaStreamSynchronize(s);
    cudaFree(wtmp);
  }
  if (wrc) return fail(PO_ERR_CUDA, "weight quantisation / tensor-map encode failed");

  // ---- activation arena (hybrid prefill: full-length hidden/qkv, chunk-bounded MLP intermediate)
  const int xcols = h > ctxc ? h : ctxc;
  const long long chunk_rows = c.chunk < T ? c.chunk : T;
  if (dalloc(e, &e->resid, (size_t)T * h * 4, &e->arena_bytes) ||
      dalloc(e, &e->xn, (size_t)T * xcols * 2, &e->arena_bytes) ||
      dalloc(e, &e->qkv, (size_t)T * qkvc * 2, &e->arena_bytes) ||
      dalloc(e, &e->xg, (size_t)T * h * 2, &e->arena_bytes) ||
      dalloc(e, &e->ss_attn, (size_t)T * (h / 128) * 4, &e->arena_bytes) ||
      dalloc(e, &e->ss_mlp, (size_t)T * (h / 128) * 4, &e->arena_bytes) ||
      dalloc(e, &e->act, (size_t)chunk_rows * I * 2, &e->arena_bytes) ||
      dalloc(e, &e->rope, (size_t)T * (c.head_dim / 2) * sizeof(float2), &e->arena_bytes))
    return fail(PO_ERR_CUDA, "arena allocation failed");
  if (f8 && (dalloc(e, &e->xg8, (size_t)T * h, &e->arena_bytes) ||
             dalloc(e, &e->ctx8, (size_t)T * ctxc, &e->arena_bytes) ||
             dalloc(e, &e->act8, (size_t)chunk_rows * I, &e->arena_bytes) ||
             dalloc(e, &e->xg_s, (size_t)T * 4, &e->arena_bytes) ||
             dalloc(e, &e->ctx_s, (size_t)T * 4, &e->arena_bytes) ||
             dalloc(e, &e->act_s, (size_t)chunk_rows * 4, &e->arena_bytes)))
    return fail(PO_ERR_CUDA, "FP8 arena allocation failed");
  if (f8) {  // rows past a launch's M are read by its last tile: keep them finite (zero codes)
    cudaMemsetAsync(e->xg8, 0, (size_t)T * h, s);
    cudaMemsetAsync(e->ctx8, 0, (size_t)T * ctxc, s);
    cudaMemsetAsync(e->act8, 0, (size_t)chunk_rows * I, s);
  }
  cudaMemsetAsync(e->qkv, 0, (size_t)T * qkvc * 2, s);
  {
    // split-KV workspace: largest need over query lengths that trigger splitting, at n_total = max_tokens
    size_t ws = 0;
    // (every query length: the need is splits x n_q, largest at the top of each constant-split band)
    for (int nq = 1; nq <= 148 * 128 && nq <= T; ++nq)
      ws = std::max(ws, po::attention_workspace_bytes((int)T, (int)T - nq, c.n_heads, c.n_kv_heads));
    e->attn_ws_bytes = ws;
    if (ws && dalloc(e, &e->attn_ws, ws, &e->workspace_bytes))
      return fail(PO_ERR_CUDA, "attention workspace failed");
    // split-K workspace: largest need over the layer GEMM shapes for every M (the split count is constant inside a
    // 128- or 256-row band, so the need peaks at band tops; every M is checked). Launchers also run unsplit when a
    // plan would exceed split_ws_bytes.
    size_t gw = 0;
    auto ws_of = f8 ? po::gemm_split_ws_bytes_f8 : po::gemm_split_ws_bytes;
    for (int m = 1; m <= 148 * 256 && m <= T; ++m) {
      gw = std::max(gw, ws_of(m, qkvc, h));
      gw = std::max(gw, ws_of(m, h, ctxc));
      gw = std::max(gw, ws_of(m, 2 * I, h));
      gw = std::max(gw, ws_of(m, h, I));
    }
    e->gemm_ws_bytes = gw;
    if (gw && dalloc(e, &e->gemm_ws, gw, &e->workspace_bytes)) return fail(PO_ERR_CUDA, "GEMM workspace failed");
    if (dalloc(e, &e->lm_ticket, 4, &e->workspace_bytes)) return fail(PO_ERR_CUDA, "LM head counter failed");
    cudaMemsetAsync(e->lm_ticket, 0, 4, s);
    if (!f8 && chunk_rows >= 512) {  // fused MLP: the act buffer is a two-piece ring
      e->mlp_piece_max = (int)(chunk_rows / 2);
      const size_t nc = po::mlp_counter_ints(T, e->mlp_piece_max);
      if (dalloc(e, &e->mlp_cnt, nc * 4, &e->workspace_bytes) || dalloc(e, &e->mlp_ticket, 4, &e->workspace_bytes) ||
          dalloc(e, &e->mlp_next, 4, &e->workspace_bytes))
        return fail(PO_ERR_CUDA, "MLP counters failed");
      cudaMemsetAsync(e->mlp_cnt, 0, nc * 4, s);
      cudaMemsetAsync(e->mlp_ticket, 0, 4, s);
      cudaMemsetAsync(e->mlp_next, 0, 4, s);
    }
    if (!f8) {  // stream-K short-launch GEMMs
      if (dalloc(e, &e->sk_ws, po::gemm_sk_ws_bytes(), &e->workspace_bytes) ||
          dalloc(e, &e->sk_flags, po::gemm_sk_flag_bytes(), &e->workspace_bytes))
        return fail(PO_ERR_CUDA, "stream-K workspace failed");
      cudaMemsetAsync(e->sk_flags, 0, po::gemm_sk_flag_bytes(), s);
    }
    if (!f8) {  // streaming kernel (requests of <= 256 miss rows): partials at M = 256 for the four layer GEMMs
      size_t sw = 0, nf = 0;
      const int shapes[4][2] = {{qkvc, h}, {h, ctxc}, {2 * I, h}, {h, I}};
      for (auto& sh : shapes) {
        sw = std::max(sw, po::stream_ws_bytes(256, sh[0], sh[1]));
        nf = std::max(nf, po::stream_flag_count(sh[0], sh[1]));
      }
      e->stream_ws_bytes = sw;
      e->stream_n_flags = nf;
      if (dalloc(e, &e->stream_ws, sw, &e->workspace_bytes) ||
          dalloc(e, &e->stream_flags, nf * 4, &e->workspace_bytes) ||
          dalloc(e, &e->stream_bar, 8, &e->workspace_bytes))
        return fail(PO_ERR_CUDA, "streaming workspace failed");
      cudaMemsetAsync(e->stream_flags, 0, nf * 4, s);
      cudaMemsetAsync(e->stream_bar, 0, 8, s);
    }
  }
  const long long max_blocks = T / c.block_tokens + 1;
  for (int i = 0; i < po_engine::STAGE_RING; ++i)
    if (dalloc(e, &e->ring_d_slots[i], (size_t)max_blocks * 4, &e->arena_bytes) ||
        dalloc(e, &e->ring_d_kvslot[i], (size_t)max_blocks * 4, &e->arena_bytes) ||
        halloc(&e->ring_h_slots[i], (size_t)max_blocks * 4) || halloc(&e->ring_h_kvslot[i], (size_t)max_blocks * 4) ||
        halloc(&e->ring_h_tokens[i], (size_t)T * 4) || halloc(&e->ring_h_allowed[i], (size_t)c.vocab * 4) ||
        halloc(&e->ring_h_logits[i], (size_t)c.vocab * 4) || halloc(&e->ring_h_probs[i], (size_t)c.vocab * 4) ||
        halloc(&e->ring_h_argmax[i], 16) ||
        cudaEventCreateWithFlags(&e->ring_ev[i], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreate(&e->ring_ev0[i]) != cudaSuccess || cudaEventCreate(&e->ring_ev1[i]) != cudaSuccess)
      return fail(PO_ERR_CUDA, "staging ring allocation failed");
  if (dalloc(e, &e->d_tokens, (size_t)T * 4, &e->arena_bytes) ||
      dalloc(e, &e->d_allowed, (size_t)c.vocab * 4, &e->arena_bytes) ||
      dalloc(e, &e->d_logits, (size_t)c.vocab * 4, &e->arena_bytes) ||
      dalloc(e, &e->d_probs, (size_t)c.vocab * 4, &e->arena_bytes) ||
      dalloc(e, &e->d_argmax, 16, &e->arena_bytes))
    return fail(PO_ERR_CUDA, "staging allocation failed");
  {
    const std::vector<float> inv = rope_inv_freq(c);
    const int half = c.head_dim / 2;
    std::vector<float2> table((size_t)T * half);
    for (long long p = 0; p < T; ++p)
      for (int i = 0; i < half; ++i) {
        const float ang = static_cast<float>(p) * inv[i];  // fp32 product, as in HF (inv_freq @ positions)
        table[(size_t)p * half + i] = make_float2(static_cast<float>(std::cos(static_cast<double>(ang))),
                                                  static_cast<float>(std::sin(static_cast<double>(ang))));
      }
    if (cudaMemcpyAsync(e->rope, table.data(), table.size() * sizeof(float2), cudaMemcpyHostToDevice, s) !=
        cudaSuccess)
      return fail(PO_ERR_CUDA, "rope table upload failed");
    cudaStreamSynchronize(s);
  }
  {
    // L2-resident MLP intermediate: when the chunk buffer (gate/up output = down input) fits the persisting L2
    // carve-out (chunk <= ~2800 rows for Llama-8B), pin it with a persisting access-policy window so it never
    // streams to HBM; the weight streams otherwise evict it (ncu: profiles/r1_mlp_l2_summary.md).
    // PO_ACT_PERSIST=0 disables, =1 forces a (partial) window.
    const char* v = getenv("PO_ACT_PERSIST");
    const size_t act_bytes = (size_t)chunk_rows * I * 2;
    int dev = 0, max_persist = 0, max_window = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev);
    const bool on = v ? v[0] == '1' : (max_persist > 0 && act_bytes <= (size_t)max_persist);
    if (on && max_window > 0) {
      const size_t win = std::min(act_bytes, (size_t)max_window);
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min(win, (size_t)max_persist));
      cudaStreamAttrValue at = {};
      at.accessPolicyWindow.base_ptr = e->act;
      at.accessPolicyWindow.num_bytes = win;
      at.accessPolicyWindow.hitRatio = std::min(1.0f, (float)max_persist / (float)win);
      at.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      at.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &at);
      e->act_persist = true;
    }
  }
  if (po::make_tmap_a(&e->map_xn, e->xn, h, T, h) || po::make_tmap_a(&e->map_ctx, e->xn, ctxc, T, ctxc) ||
      po::make_tmap_a(&e->map_xg, e->xg, h, T, h) ||
      po::make_tmap_a(&e->map_act, e->act, I, chunk_rows, I))
    return fail(PO_ERR_CUDA, "activation tensor-map encode failed");
  if (f8 && (po::make_tmap_a_f8(&e->map_xg8, e->xg8, h, T, h) || po::make_tmap_a_f8(&e->map_ctx8, e->ctx8, ctxc, T, ctxc) ||
             po::make_tmap_a_f8(&e->map_act8, e->act8, I, chunk_rows, I)))
    return fail(PO_ERR_CUDA, "FP8 activation tensor-map encode failed");

  // ---- prefix pool: explicit size, or a profile run: what remains after weights + arena
  if (cudaStreamSynchronize(s) != cudaSuccess) return fail(PO_ERR_CUDA, "init kernels failed");
  const int64_t bb = e->block_bytes();
  if (c.pool_blocks >= 0) {
    e->pool_blocks = c.pool_blocks;
  } else {
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    const double frac = (c.pool_mem_fraction > 0 && c.pool_mem_fraction <= 1) ? c.pool_mem_fraction : 0.9;
    const int64_t reserve = 2ll << 30;  // headroom for the CUDA context, cuBLAS/torch workspaces
    const int64_t avail = (int64_t)free_b > reserve ? (int64_t)((free_b - reserve) * frac) : 0;
    e->pool_blocks = avail / bb;
  }
  if (e->pool_blocks > 0 && dalloc(e, &e->pool, (size_t)(e->pool_blocks * bb), &e->pool_bytes))
    return fail(PO_ERR_CUDA, "prefix pool allocation failed");
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  e->free_after = (int64_t)free_b;
  *out = e;
  return PO_OK;
}

int po_engine_info(po_engine* e, int64_t* out, int32_t n) {
  if (!e || !out) return set_error(PO_ERR_ARG, "po_engine_info: null argument");
  const int64_t v[8] = {e->pool_blocks, e->weight_bytes, e->arena_bytes, e->pool_bytes, e->block_bytes(),
                        e->cfg.max_tokens, e->free_after, e->workspace_bytes};
  for (int i = 0; i < n && i < 8; ++i) out[i] = v[i];
  return PO_OK;
}

int po_last_service_ms(po_engine* e, float* ms) {
  if (!e || !ms) return set_error(PO_ERR_ARG, "po_last_service_ms: null argument");
  *ms = e->last_ms;
  if (getenv("PO_ENQUEUE_TIMING")) fprintf(stderr, "enqueue %.3f ms service %.3f ms\n", e->last_enqueue_ms, e->last_ms);
  return PO_OK;
}

int po_pool_evict(po_engine* e, const int32_t* slots, int32_t n) {
  if (!e) return set_error(PO_ERR_ARG, "po_pool_evict: null engine");
  for (int i = 0; i < n; ++i)
    if (slots[i] < 0 || slots[i] >= e->pool_blocks)
      return set_error(PO_ERR_POOL, "po_pool_evict: slot %d out of range [0, %lld)", slots[i],
                       (long long)e->pool_blocks);
  return PO_OK;
}

int po_load_weight(po_engine* e, int32_t kind, int32_t layer, const void* host, int64_t nelem) {
  if (!e || !host) return set_error(PO_ERR_ARG, "po_load_weight: null argument");
  const po_model_cfg& c = e->cfg;
  const int h = c.hidden, I = c.intermediate;
  const int qrows = c.n_heads * c.head_dim, kvrows = c.n_kv_heads * c.head_dim;
  if (((kind >= 1 && kind <= 9) || kind == 12) && (layer < 0 || layer >= c.num_layers))
    return set_error(PO_ERR_ARG, "po_load_weight: layer %d out of range", layer);
  cudaSetDevice(e->device);
  void* dst = nullptr;
  int64_t expect = 0;
  bool norm = false;
  auto& ly = e->layers[((kind >= 1 && kind <= 9) || kind == 12) ? layer : 0];
  switch (kind) {
    case 0: dst = e->embed; expect = (int64_t)c.vocab * h; break;
    case 1: dst = ly.attn_norm; expect = h; norm = true; break;
    case 2: dst = ly.wqkv; expect = (int64_t)qrows * h; break;
    case 3: dst = ly.wqkv + (size_t)qrows * h; expect = (int64_t)kvrows * h; break;
    case 4: dst = ly.wqkv + (size_t)(qrows + kvrows) * h; expect = (int64_t)kvrows * h; break;
    case 5: dst = ly.wo; expect = (int64_t)h * qrows; break;
    case 6: dst = ly.mlp_norm; expect = h; norm = true; break;
    case 7:
    case 8: expect = (int64_t)I * h; break;
    case 9: dst = ly.wdown; expect = (int64_t)h * I; break;
    case 10: dst = e->final_norm; expect = h; norm = true; break;
    case 11: dst = e->lm_head; expect = (int64_t)c.vocab * h; break;
    case 12:
      if (!c.qkv_bias) return set_error(PO_ERR_ARG, "po_load_weight: model has no qkv bias");
      dst = ly.bqkv; expect = (int64_t)e->qkv_cols(); norm = true; break;
    default: return set_error(PO_ERR_ARG, "po_load_weight: unknown kind %d", kind);
  }
  if (nelem != expect)
    return set_error(PO_ERR_ARG, "po_load_weight: kind %d expects %lld elements, got %lld", kind, (long long)expect,
                     (long long)nelem);
  if (e->fp8() && (kind == 2 || kind == 3 || kind == 4 || kind == 5 || kind == 7 || kind == 8 || kind == 9)) {
    // FP8 engine: the bf16 rows are quantised per row on the device into the E4M3 copy (+ scales)
    int rows = 0, cols = h;
    uint8_t* q = nullptr;
    float* sc = nullptr;
    switch (kind) {
      case 2: rows = qrows; q = ly.q_qkv; sc = ly.s_qkv; break;
      case 3: rows = kvrows; q = ly.q_qkv + (size_t)qrows * h; sc = ly.s_qkv + qrows; break;
      case 4: rows = kvrows; q = ly.q_qkv + (size_t)(qrows + kvrows) * h; sc = ly.s_qkv + qrows + kvrows; break;
      case 5: rows = h; cols = qrows; q = ly.q_o; sc = ly.s_o; break;
      case 9: rows = h; cols = I; q = ly.q_down; sc = ly.s_down; break;
      default: rows = I; break;  // 7 / 8: gate or up, interleaved below
    }
    __nv_bfloat16* tmp = nullptr;
    uint8_t* tq = nullptr;
    float* ts = nullptr;
    int rc = 0;
    if (cudaMalloc(&tmp, (size_t)rows * cols * 2) != cudaSuccess ||
        cudaMalloc(&tq, (size_t)rows * cols) != cudaSuccess || cudaMalloc(&ts, (size_t)rows * 4) != cudaSuccess ||
        cudaMemcpy(tmp, host, (size_t)rows * cols * 2, cudaMemcpyHostToDevice) != cudaSuccess ||
        po::quantize_rows_e4m3(tmp, cols, rows, cols, tq, cols, ts, nullptr) != 0 ||
        cudaDeviceSynchronize() != cudaSuccess)
      rc = -1;
    if (!rc && (kind == 7 || kind == 8)) {
      // interleave 16-row groups into the fused gate/up layout, gate first (rows and their scales)
      const int off = kind == 7 ? 0 : 16;
      for (int g = 0; g < I / 16 && !rc; ++g)
        if (cudaMemcpy(ly.q_gu + ((size_t)g * 32 + off) * h, tq + (size_t)g * 16 * h, (size_t)16 * h,
                       cudaMemcpyDeviceToDevice) != cudaSuccess ||
            cudaMemcpy(ly.s_gu + (size_t)g * 32 + off, ts + (size_t)g * 16, 16 * 4, cudaMemcpyDeviceToDevice) !=
                cudaSuccess)
          rc = -1;
    } else if (!rc) {
      if (cudaMemcpy(q, tq, (size_t)rows * cols, cudaMemcpyDeviceToDevice) != cudaSuccess ||
          cudaMemcpy(sc, ts, (size_t)rows * 4, cudaMemcpyDeviceToDevice) != cudaSuccess)
        rc = -1;
    }
    cudaFree(tmp);
    cudaFree(tq);
    cudaFree(ts);
    return rc ? set_error(PO_ERR_CUDA, "po_load_weight: FP8 quantisation / copy failed") : PO_OK;
  }
  if (kind == 7 || kind == 8) {
    // interleave into the fused gate/up layout: 16-row groups, gate first
    const __nv_bfloat16* src = static_cast<const __nv_bfloat16*>(host);
    const int off = kind == 7 ? 0 : 16;
    for (int g = 0; g < I / 16; ++g)
      if (cudaMemcpy(ly.wgu + ((size_t)g * 32 + off) * h, src + (size_t)g * 16 * h, (size_t)16 * h * 2,
                     cudaMemcpyHostToDevice) != cudaSuccess)
        return set_error(PO_ERR_CUDA, "po_load_weight: copy failed");
    return PO_OK;
  }
  if (cudaMemcpy(dst, host, (size_t)nelem * (norm ? 4 : 2), cudaMemcpyHostToDevice) != cudaSuccess)
    return set_error(PO_ERR_CUDA, "po_load_weight: copy failed");
  return PO_OK;
}

namespace {
// MLP row pieces of a layer (each <= chunk rows; the act buffer holds one piece). The pair GEMMs run 256 x 256 tiles
// over P = SMs / 2 pairs, so a piece of b 256-row blocks costs ceil(b * tiles_per_block / P) waves of each GEMM, a wave
// taking time proportional to K. Equal row pieces (20,000 rows -> 3 x 6,667) round every piece up to whole blocks
// and whole waves; here the ceil(rows / chunk) pieces take whole 256-row blocks (the last one the remainder rows)
// split to minimise the summed wave cost of gate/up (K = hidden, 2I / 256 tiles per block) and down (K = I,
// hidden / 256 tiles per block): 20,000 rows -> 4,352 + 7,936 + 7,712 (gate/up 26 + 47 + 47 waves instead of
// 3 x 41). PO_PIECE_PLAN=0 keeps the equal pieces. Returns the piece row counts in launch order.
void plan_mlp_pieces(int rows, int chunk, int hidden, int inter, int pairs, std::vector<int>& out) {
  out.clear();
  if (rows <= 0) return;
  const int n_pieces = (rows + chunk - 1) / chunk;
  static int mode = -1;
  if (mode < 0) mode = (getenv("PO_PIECE_PLAN") && getenv("PO_PIECE_PLAN")[0] == '0') ? 0 : 1;
  const int B = (rows + 255) / 256;
  const int maxb = chunk / 256;
  if (mode == 0 || n_pieces == 1 || chunk % 256 || maxb < 1 || pairs < 1 || (long long)n_pieces * maxb < B ||
      n_pieces > 64 || B > 4096) {
    const int piece = (rows + n_pieces - 1) / n_pieces;
    for (int lo = 0; lo < rows; lo += piece) out.push_back(std::min(piece, rows - lo));
    return;
  }
  const long long tgu = 2LL * inter / 256, tdn = hidden / 256;
  auto cost = [&](int b) {
    return (long long)hidden * ((b * tgu + pairs - 1) / pairs) + (long long)inter * ((b * tdn + pairs - 1) / pairs);
  };
  // best[k][u]: least cost of k pieces covering u blocks; pick[k][u]: the last piece's blocks
  const long long INF = (1LL << 62);
  std::vector<long long> best((size_t)(n_pieces + 1) * (B + 1), INF);
  std::vector<int> pick((size_t)(n_pieces + 1) * (B + 1), 0);
  best[0] = 0;
  for (int k = 1; k <= n_pieces; ++k)
    for (int u = 1; u <= B; ++u)
      for (int b = 1; b <= maxb && b <= u; ++b) {
        const long long prev = best[(size_t)(k - 1) * (B + 1) + u - b];
        if (prev == INF) continue;
        const long long c = prev + cost(b);
        if (c < best[(size_t)k * (B + 1) + u]) {
          best[(size_t)k * (B + 1) + u] = c;
          pick[(size_t)k * (B + 1) + u] = b;
        }
      }
  std::vector<int> blocks;
  for (int k = n_pieces, u = B; k > 0; --k) {
    const int b = pick[(size_t)k * (B + 1) + u];
    blocks.push_back(b);
    u -= b;
  }
  // whole blocks first, the remainder rows in the last piece
  int done = 0;
  for (size_t i = 0; i < blocks.size(); ++i) {
    const int r = i + 1 < blocks.size() ? blocks[i] * 256 : rows - done;
    out.push_back(r);
    done += r;
  }
}

// Validate a request and stage its block table; returns n_c (computed-from prefix) or a negative status.
int stage_request(po_engine* e, int32_t n, int32_t n_cached, int32_t n_allowed, const int32_t* pool_block_ids,
                  int32_t n_blocks, int* n_admit_out) {
  const po_model_cfg& c = e->cfg;
  if (n <= 0) return set_error(PO_ERR_ARG, "po_prefill: empty request");
  if (n > c.max_tokens)
    return set_error(PO_ERR_CAPACITY, "po_prefill: request of %d tokens exceeds MIL %d", n, c.max_tokens);
  if (n_cached < 0 || n_cached > n || n_cached % c.block_tokens)
    return set_error(PO_ERR_ARG, "po_prefill: need 0 <= n_cached <= n, block aligned (got %d of %d)", n_cached, n);
  if (n_allowed <= 0 || n_allowed > c.vocab)
    return set_error(PO_ERR_ARG, "po_prefill: allowed list must hold 1..vocab ids (got %d)", n_allowed);
  const int bt = c.block_tokens;
  if (n_blocks < 0 || n_blocks > n / bt) return set_error(PO_ERR_ARG, "po_prefill: n_blocks %d > n/bt", n_blocks);
  if (n_cached / bt > n_blocks || (n_blocks > 0 && !pool_block_ids))
    return set_error(PO_ERR_ARG, "po_prefill: cached blocks need pool slots");
  // next staging-ring entry: wait until the forward that last used it (and its table copies) has completed
  const int ri = e->ring_next;
  if (cudaEventSynchronize(e->ring_ev[ri]) != cudaSuccess)
    return set_error(PO_ERR_CUDA, "po_prefill: an earlier forward failed: %s", cudaGetErrorString(cudaGetLastError()));
  e->h_slots = e->ring_h_slots[ri];
  e->h_kvslot = e->ring_h_kvslot[ri];
  e->d_slots = e->ring_d_slots[ri];
  e->d_kvslot = e->ring_d_kvslot[ri];
  e->h_tokens = e->ring_h_tokens[ri];
  e->h_allowed = e->ring_h_allowed[ri];
  e->h_logits = e->ring_h_logits[ri];
  e->h_probs = e->ring_h_probs[ri];
  e->h_argmax = e->ring_h_argmax[ri];
  e->cur_ring = ri;
  // a fully cached request still recomputes its last token to produce logits
  const int n_c = n_cached < n ? n_cached : n - 1;
  const int cached_blocks = (n_c + bt - 1) / bt;
  int n_admit = 0;
  for (int b = 0; b <= n / bt; ++b) e->h_kvslot[b] = -1;
  // a slot may appear once per request: two admitted blocks on one slot race in the QKV epilogue, and an admitted
  // block on a cached block's slot would overwrite keys this forward's attention still reads
  if ((int64_t)e->slot_stamp.size() != e->pool_blocks) e->slot_stamp.assign((size_t)e->pool_blocks, 0u);
  if (++e->stamp_gen == 0) {
    std::fill(e->slot_stamp.begin(), e->slot_stamp.end(), 0u);
    e->stamp_gen = 1;
  }
  for (int b = 0; b < n_blocks; ++b) {
    const int slot = pool_block_ids[b];
    if (b < n_cached / bt) {
      if (slot < 0 || slot >= e->pool_blocks)
        return set_error(PO_ERR_POOL, "po_prefill: cached block %d has invalid slot %d", b, slot);
      if (b < cached_blocks) e->h_slots[b] = slot;
    } else if (slot >= 0) {
      if (slot >= e->pool_blocks) return set_error(PO_ERR_POOL, "po_prefill: admit slot %d out of range", slot);
      e->h_kvslot[b] = slot;
      ++n_admit;
    } else {
      continue;
    }
    if (e->slot_stamp[slot] == e->stamp_gen)
      return set_error(PO_ERR_POOL, "po_prefill: pool slot %d named twice in one request (block %d)", slot, b);
    e->slot_stamp[slot] = e->stamp_gen;
  }
  *n_admit_out = n_admit;
  return n_c;
}

// 2-CTA pair GEMM for M > 128 (256-row pair tiles), 1-CTA 128-row tiles below
bool bounded_a_enabled();

// x / ldx: the activation buffer behind `a`. A launch whose rows stop short of its A tile (short miss suffixes, the
// last layer's final row) gets a map bounded at its last row, so the padding rows of the 128-row boxes are
// zero-filled by TMA instead of being read from memory (for M = 1 that is 127 wasted rows per weight tile).
int gemm(const CUtensorMap& a, const void* x, long long ldx, const CUtensorMap& b1, const CUtensorMap& b2,
         const CUtensorMap& b3, int epi, const po::GemmArgs& g, cudaStream_t s) {
  if (po::gemm_swap_enabled() && g.M <= 256) {  // short launches: weight as the MMA's M operand
    if (g.sk_ws && po::gemm_sk_enabled(epi)) {  // stream-K: one round, in-kernel fix-up
      const int rc = po::gemm_launch_sk(b2, x, ldx, epi, g, s);
      if (rc != 1) return rc;
    }
    const int rc = po::gemm_launch_swap(b2, x, ldx, epi, g, s);
    if (rc != 1) return rc;
  }
  const CUtensorMap* am = &a;
  CUtensorMap bounded;
  if (g.M % 128 != 0 && bounded_a_enabled()) {
    if (po::make_tmap_a(&bounded, x, ldx, (long long)g.a_row0 + g.M, g.K)) return -2;
    am = &bounded;
  }
  return po::gemm_use_pair(g.M) ? po::gemm_launch_pair(*am, b2, epi, g, s, &b3) : po::gemm_launch(*am, b1, epi, g, s);
}

// weight_fp8: quantise the launch's A rows [a_row0, a_row0 + M) per row (E4M3 + scale), then the W8A8 pair GEMM
// with the weight's per-channel scales. Two launches.
int gemm8(const CUtensorMap& a8, const __nv_bfloat16* x, long long ldx, uint8_t* x8, float* xs, const CUtensorMap& b8,
          const float* bs, int epi, po::GemmArgs g, cudaStream_t s) {
  if (int rc = po::quantize_rows_e4m3(x + (size_t)g.a_row0 * ldx, ldx, g.M, g.K, x8 + (size_t)g.a_row0 * g.K, g.K,
                                      xs + g.a_row0, s))
    return rc;
  g.a_scale = xs + g.a_row0;
  g.b_scale = bs;
  return po::gemm_launch_pair_f8(a8, b8, epi, g, s);
}

// PO_BOUNDED_A=0 keeps the whole-buffer activation maps (A/B runs)
bool bounded_a_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* v = getenv("PO_BOUNDED_A");
    on = (v && v[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

// PO_POOL_DIRECT=0 gathers the cached K/V into the layer buffer before attention (A/B runs)
bool pool_direct_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* v = getenv("PO_POOL_DIRECT");
    on = (v && v[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

enum KClass { KC_EMBED = 0, KC_NORM, KC_GATHER, KC_QKV, KC_SCATTER, KC_ATTN, KC_O, KC_GATE_UP, KC_DOWN, KC_LM_HEAD,
              KC_STREAM, KC_MLP, KC_COUNT };

// PO_STREAM=1 runs prefix hits' layer GEMMs through the persistent streaming kernel (stream.cu). Off by default:
// its mainloop streams weights faster than the per-GEMM launches, but the in-kernel split-tile fix-up is
// latency-bound with four epilogue warps per SM, so the forward is slower.
bool stream_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* v = getenv("PO_STREAM");
    on = (v && v[0] == '1') ? 1 : 0;
  }
  return on == 1;
}

// The hybrid-prefill forward on device-resident inputs; asynchronous on stream s.
int forward(po_engine* e, const uint32_t* d_tok_miss, int n, int n_c, int n_admit, const int* d_allowed,
            int n_allowed, float* d_logits, float* d_probs, int* d_argmax, cudaStream_t s) {
  const po_model_cfg& c = e->cfg;
  const int bt = c.block_tokens;
  const int n_miss = n - n_c;
  const int cached_blocks = (n_c + bt - 1) / bt;
  const int h = c.hidden, I = c.intermediate, L = c.num_layers;
  const int qkvc = e->qkv_cols(), ctxc = e->ctx_cols(), kvd = e->kv_dim();
  const int kv_col0 = c.n_heads * c.head_dim;
  const bool f8 = e->fp8();
  int launches = 0;
  auto mark = [&](int cls, bool begin) {
    if (!e->profiling) return;
    if (begin) {
      if (e->prof_used >= (int)e->prof_events.size()) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        e->prof_events.push_back({a, b});
        e->prof_class.push_back(0);
      }
      e->prof_class[e->prof_used] = cls;
      cudaEventRecord(e->prof_events[e->prof_used].first, s);
    } else {
      cudaEventRecord(e->prof_events[e->prof_used].second, s);
      ++e->prof_used;
    }
  };
  if (cached_blocks) cudaMemcpyAsync(e->d_slots, e->h_slots, (size_t)cached_blocks * 4, cudaMemcpyHostToDevice, s);
  if (n_admit) cudaMemcpyAsync(e->d_kvslot, e->h_kvslot, (size_t)(n / bt + 1) * 4, cudaMemcpyHostToDevice, s);

  // RMSNorm is folded across the GEMMs (GemmArgs): producers (embedding, residual epilogues) write
  // xg = bf16(resid . gamma_next) and per-segment sums of squares; consumers scale rows by 1/rms.
  const int nseg = h / 128;
  mark(KC_EMBED, true);
  po::launch_embed_norm(d_tok_miss, n_miss, e->embed, c.vocab, h, e->layers[0].attn_norm, e->resid, e->xg,
                        e->ss_attn, s);
  mark(KC_EMBED, false);
  ++launches;
  auto norm_in = [&](po::GemmArgs& g, const float* ss) {
    g.ss_in = ss; g.ss_nseg = nseg; g.norm_eps = c.rms_eps; g.norm_dim = h;
  };
  auto norm_out = [&](po::GemmArgs& g, __nv_bfloat16* xg, const float* gamma, float* ss) {
    g.xg_out = xg; g.ldxg = h; g.g_next = gamma; g.ss_out = ss; g.ss_nseg = nseg;
  };
  int rc = 0;
  // Prefix hits (n_miss <= 256): the layer GEMMs are weight streams and run as phases of the persistent streaming
  // kernel (stream.cu), batched O -> gate/up -> down -> next QKV between two attention launches. Larger requests run
  // one tcgen05 GEMM launch per matrix.
  const bool streaming = !f8 && n_miss <= 256 && e->stream_ws && stream_enabled();
  po::StreamArgs sa{};
  auto flush = [&]() -> int {
    if (!sa.nph) return 0;
    sa.ws = e->stream_ws; sa.ws_bytes = e->stream_ws_bytes; sa.flags = e->stream_flags;
    sa.n_flags = e->stream_n_flags; sa.bar = e->stream_bar; sa.bar_base = e->stream_bar_base; sa.tag = e->stream_tag;
    mark(KC_STREAM, true);
    const int r = po::stream_launch(sa, s);
    mark(KC_STREAM, false);
    if (!r) {
      e->stream_bar_base += (unsigned long long)sa.nph * 2 * po::stream_pairs();
      ++e->stream_tag;
      ++launches;
    }
    sa.nph = 0;
    return r;
  };
  // one layer GEMM: a streaming phase, or its own launch(es)
  auto run_gemm = [&](int cls, const CUtensorMap& amap, const void* x, long long ldx, const CUtensorMap& b1,
                      const CUtensorMap& b2, const CUtensorMap& b3, int epi, const po::GemmArgs& g,
                      const CUtensorMap& a8, uint8_t* x8, float* xs, const CUtensorMap& bq, const float* bsc) -> int {
    if (g.M <= 0) return 0;
    if (streaming) {
      po::StreamPhase& ph = sa.ph[sa.nph];
      if (po::make_tmap_a(&ph.a, x, ldx, (long long)g.a_row0 + g.M, g.K)) return -2;
      ph.b = b2; ph.g = g; ph.epi = epi;
      return ++sa.nph == po::STREAM_MAX_PHASES ? flush() : 0;
    }
    mark(cls, true);
    po::GemmArgs gk = g;
    // stream-K for short requests (every layer GEMM a weight stream: prefix hits, short prompts); a long request's
    // short launches (MLP chunk tails, the last layer's final row) keep the split-K kernels, so a result does not
    // depend on the MLP chunk size
    if (n_miss <= 256) { gk.sk_ws = e->sk_ws; gk.sk_flags = e->sk_flags; gk.sk_epoch = ++e->sk_epoch; }
    int r = f8 ? gemm8(a8, static_cast<const __nv_bfloat16*>(x), ldx, x8, xs, bq, bsc, epi, g, s)
               : gemm(amap, x, ldx, b1, b2, b3, epi, gk, s);
    mark(cls, false);
    launches += f8 ? 2 : 1;
    return r;
  };
  auto qkv_gemm = [&](int l) -> int {
    auto& ly = e->layers[l];
    po::GemmArgs g{};
    g.M = n_miss; g.N = qkvc; g.K = h;
    g.out = e->qkv + (size_t)n_c * qkvc; g.ldo = qkvc;
    g.rope = e->rope; g.pos_offset = n_c; g.rope_cols = (c.n_heads + c.n_kv_heads) * c.head_dim;
    g.split_ws = e->gemm_ws; g.split_ws_bytes = e->gemm_ws_bytes;
    g.bias = ly.bqkv;
    if (n_admit) {  // suffix-block admission: the QKV epilogue also stores the admitted rows' K/V into the pool
      g.kv_slot = e->d_kvslot; g.kv_pool = e->pool; g.pool_layers = L; g.pool_layer = l;
      g.kv_col0 = kv_col0; g.kv_dim = kvd;
    }
    norm_in(g, e->ss_attn);
    return run_gemm(KC_QKV, e->map_xg, e->xg, h, ly.map_qkv, ly.map2_qkv, ly.map3_qkv, po::EPI_QKV_ROPE, g,
                    e->map_xg8, e->xg8, e->xg_s, ly.f8_qkv, ly.s_qkv);
  };
  rc |= qkv_gemm(0);
  for (int l = 0; l < L && !rc; ++l) {
    auto& ly = e->layers[l];
    const float* gamma_next_layer = l + 1 < L ? e->layers[l + 1].attn_norm : e->final_norm;
    rc |= flush();  // this layer's QKV (and the previous layer's tail) complete before attention
    // cached prefix K/V: read by attention straight from the pool (pool-direct), or gathered into qkv first
    const bool pool_direct = n_c > 0 && pool_direct_enabled() && bt == 16;
    if (n_c > 0 && !pool_direct) {
      mark(KC_GATHER, true);
      po::launch_kv_gather(e->pool, e->d_slots, n_c, l, L, bt, kvd, e->qkv, qkvc, kv_col0, s);
      mark(KC_GATHER, false);
      ++launches;
    }
    // the last layer only needs the final row's output (the LM head reads nothing else); its K/V rows
    // were computed (and admitted to the pool) above
    const bool last_only = c.last_row_only && l == L - 1 && n_miss > 1;
    const int q_first = last_only ? n - 1 : n_c;       // first query position this layer computes
    const int rows = n - q_first;                      // query rows of attention / O / MLP
    const int row0 = q_first - n_c;                    // their offset inside the miss rows
    mark(KC_ATTN, true);
    // whole cached blocks come from the pool (a fully cached request's last block too: its K/V are in the pool)
    po::AttnPool ap{e->pool, e->d_slots, pool_direct ? cached_blocks * bt : 0, (int)e->pool_blocks, L, l, kvd, bt};
    rc |= po::attention_run(e->qkv, qkvc, n, q_first, c.n_heads, c.n_kv_heads, e->xn, ctxc, s, e->attn_ws,
                            e->attn_ws_bytes, pool_direct ? &ap : nullptr);
    mark(KC_ATTN, false);
    ++launches;
    po::GemmArgs go{};
    go.M = rows; go.N = h; go.K = ctxc;
    go.resid = e->resid + (size_t)row0 * h; go.ldr = h; go.split_ws = e->gemm_ws; go.split_ws_bytes = e->gemm_ws_bytes;
    norm_out(go, e->xg + (size_t)row0 * h, ly.mlp_norm, e->ss_mlp + (size_t)row0 * nseg);
    rc |= run_gemm(KC_O, e->map_ctx, e->xn, ctxc, ly.map_o, ly.map2_o, ly.map3_o, po::EPI_RESID_F32, go,
                   e->map_ctx8, e->ctx8, e->ctx_s, ly.f8_o, ly.s_o);
    const int mlp_rows = n_miss - row0;
    if (!rc && e->mlp_cnt && mlp_rows > 256 && po::mlp_fused_enabled()) {
      // the whole MLP of the layer in one launch: gate/up and down tiles of balanced row pieces, the intermediate in
      // the L2-pinned two-piece ring (mlp.cu)
      po::MlpArgs ma{};
      ma.rows = mlp_rows;
      const int npc = (mlp_rows + e->mlp_piece_max - 1) / e->mlp_piece_max;
      ma.piece = (mlp_rows + npc - 1) / npc;
      ma.cnt = e->mlp_cnt;
      ma.ticket = e->mlp_ticket;
      ma.next = e->mlp_next;
      po::GemmArgs& gu = ma.gu;
      gu.M = mlp_rows; gu.N = 2 * I; gu.K = h; gu.a_row0 = row0;
      gu.out = e->act; gu.ldo = I;
      norm_in(gu, e->ss_mlp + (size_t)row0 * nseg);
      po::GemmArgs& gd = ma.dn;
      gd.M = mlp_rows; gd.N = h; gd.K = I;
      gd.resid = e->resid + (size_t)row0 * h; gd.ldr = h;
      norm_out(gd, e->xg + (size_t)row0 * h, gamma_next_layer, e->ss_attn + (size_t)row0 * nseg);
      mark(KC_MLP, true);
      rc |= po::mlp_launch(e->map_xg, ly.map2_gu, e->map_act, ly.map2_down, ma, s);
      mark(KC_MLP, false);
      ++launches;
      if (l + 1 < L) rc |= qkv_gemm(l + 1);
      continue;
    }
    // ceil(rows / chunk) pieces planned against the GEMMs' wave quantisation (plan_mlp_pieces)
    if (e->piece_plan_rows != mlp_rows) {
      plan_mlp_pieces(mlp_rows, c.chunk, h, I, po::num_sms() / 2, e->piece_plan);
      e->piece_plan_rows = mlp_rows;
    }
    int lo = row0;
    for (size_t pi = 0; pi < e->piece_plan.size() && !rc; lo += e->piece_plan[pi], ++pi) {
      const int cr = e->piece_plan[pi];
      po::GemmArgs gu{};
      gu.M = cr; gu.N = 2 * I; gu.K = h; gu.a_row0 = lo;
      gu.out = e->act; gu.ldo = I; gu.split_ws = e->gemm_ws; gu.split_ws_bytes = e->gemm_ws_bytes;
      norm_in(gu, e->ss_mlp + (size_t)lo * nseg);
      rc |= run_gemm(KC_GATE_UP, e->map_xg, e->xg, h, ly.map_gu, ly.map2_gu, ly.map3_gu, po::EPI_SILU_MUL, gu,
                     e->map_xg8, e->xg8, e->xg_s, ly.f8_gu, ly.s_gu);
      po::GemmArgs gd{};
      gd.M = cr; gd.N = h; gd.K = I;
      gd.resid = e->resid + (size_t)lo * h; gd.ldr = h; gd.split_ws = e->gemm_ws; gd.split_ws_bytes = e->gemm_ws_bytes;
      norm_out(gd, e->xg + (size_t)lo * h, gamma_next_layer, e->ss_attn + (size_t)lo * nseg);
      rc |= run_gemm(KC_DOWN, e->map_act, e->act, I, ly.map_down, ly.map2_down, ly.map3_down, po::EPI_RESID_F32, gd,
                     e->map_act8, e->act8, e->act_s, ly.f8_down, ly.s_down);
    }
    if (l + 1 < L) rc |= qkv_gemm(l + 1);
  }
  rc |= flush();
  if (rc) return set_error(PO_ERR_CUDA, "po_prefill: kernel launch failed (%d): %s", rc,
                           cudaGetErrorString(cudaGetLastError()));
  mark(KC_LM_HEAD, true);
  po::launch_lm_head(e->resid + (size_t)(n_miss - 1) * h, h, e->final_norm, c.rms_eps, e->lm_head, d_allowed,
                     n_allowed, d_logits, d_probs, d_argmax, e->lm_ticket, s);
  mark(KC_LM_HEAD, false);
  ++launches;
  e->last_launches = launches;
  if (cudaGetLastError() != cudaSuccess) return set_error(PO_ERR_CUDA, "po_prefill: launch error");
  return PO_OK;
}

// The staged request's ring entry may be reused once everything enqueued so far (its forward, table and output
// copies) has run.
void release_ring(po_engine* e, cudaStream_t s) {
  cudaEventRecord(e->ring_ev[e->cur_ring], s);
  e->ring_next = (e->cur_ring + 1) % po_engine::STAGE_RING;
}
}  // namespace

int po_prefill_submit(po_engine* e, const uint32_t* tokens, int32_t n, int32_t n_cached, const int32_t* allowed,
                      int32_t n_allowed, const int32_t* pool_block_ids, int32_t n_blocks, int64_t* ticket,
                      void* stream) {
  if (!e || !tokens || !allowed || !ticket) return set_error(PO_ERR_ARG, "po_prefill: null argument");
  const po_model_cfg& c = e->cfg;
  for (int i = 0; i < n_allowed; ++i)
    if (allowed[i] < 0 || allowed[i] >= c.vocab)
      return set_error(PO_ERR_ARG, "po_prefill: allowed id %d out of vocab", allowed[i]);
  cudaSetDevice(e->device);
  int n_admit = 0;
  const int n_c = stage_request(e, n, n_cached, n_allowed, pool_block_ids, n_blocks, &n_admit);
  if (n_c < 0) return n_c;
  const int ri = e->cur_ring;
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : e->stream;
  const int n_miss = n - n_c;
  std::memcpy(e->h_tokens, tokens + n_c, (size_t)n_miss * 4);
  std::memcpy(e->h_allowed, allowed, (size_t)n_allowed * 4);
  e->ring_ticket[ri] = -1;  // owned by nobody until the forward is enqueued
  cudaEventRecord(e->ring_ev0[ri], s);
  cudaMemcpyAsync(e->d_tokens, e->h_tokens, (size_t)n_miss * 4, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(e->d_allowed, e->h_allowed, (size_t)n_allowed * 4, cudaMemcpyHostToDevice, s);
  const auto h0 = std::chrono::steady_clock::now();
  int rc = forward(e, e->d_tokens, n, n_c, n_admit, e->d_allowed, n_allowed, e->d_logits, e->d_probs, e->d_argmax, s);
  if (rc) {
    release_ring(e, s);
    return rc;
  }
  e->last_enqueue_ms = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - h0).count();
  cudaMemcpyAsync(e->h_logits, e->d_logits, (size_t)n_allowed * 4, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(e->h_probs, e->d_probs, (size_t)n_allowed * 4, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(e->h_argmax, e->d_argmax, 4, cudaMemcpyDeviceToHost, s);
  cudaEventRecord(e->ring_ev1[ri], s);
  release_ring(e, s);
  if (cudaGetLastError() != cudaSuccess) return set_error(PO_ERR_CUDA, "po_prefill: launch error");
  e->ring_n_allowed[ri] = n_allowed;
  e->ring_ticket[ri] = *ticket = ++e->next_ticket;
  return PO_OK;
}

namespace {
int ring_of(po_engine* e, int64_t ticket) {
  for (int i = 0; i < po_engine::STAGE_RING; ++i)
    if (e->ring_ticket[i] == ticket && ticket > 0) return i;
  return -1;
}
}  // namespace

int po_prefill_query(po_engine* e, int64_t ticket, int32_t* done) {
  if (!e || !done) return set_error(PO_ERR_ARG, "po_prefill_query: null argument");
  const int ri = ring_of(e, ticket);
  if (ri < 0) return set_error(PO_ERR_ARG, "po_prefill_query: unknown or recycled ticket %lld", (long long)ticket);
  const cudaError_t q = cudaEventQuery(e->ring_ev1[ri]);
  if (q != cudaSuccess && q != cudaErrorNotReady)
    return set_error(PO_ERR_CUDA, "po_prefill: forward failed: %s", cudaGetErrorString(q));
  *done = q == cudaSuccess;
  return PO_OK;
}

int po_prefill_wait(po_engine* e, int64_t ticket, float* out_logits, float* out_probs, int32_t* out_argmax,
                    float* service_ms) {
  if (!e) return set_error(PO_ERR_ARG, "po_prefill_wait: null engine");
  const int ri = ring_of(e, ticket);
  if (ri < 0) return set_error(PO_ERR_ARG, "po_prefill_wait: unknown or recycled ticket %lld", (long long)ticket);
  if (cudaEventSynchronize(e->ring_ev1[ri]) != cudaSuccess)
    return set_error(PO_ERR_CUDA, "po_prefill: forward failed: %s", cudaGetErrorString(cudaGetLastError()));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e->ring_ev0[ri], e->ring_ev1[ri]);
  e->last_ms = ms;
  if (service_ms) *service_ms = ms;
  const int na = e->ring_n_allowed[ri];
  if (out_logits) std::memcpy(out_logits, e->ring_h_logits[ri], (size_t)na * 4);
  if (out_probs) std::memcpy(out_probs, e->ring_h_probs[ri], (size_t)na * 4);
  if (out_argmax) *out_argmax = *e->ring_h_argmax[ri];
  e->ring_ticket[ri] = 0;  // consumed
  return PO_OK;
}

int po_prefill(po_engine* e, const uint32_t* tokens, int32_t n, int32_t n_cached, const int32_t* allowed,
               int32_t n_allowed, const int32_t* pool_block_ids, int32_t n_blocks, float* out_logits,
               float* out_probs, int32_t* out_argmax, void* stream) {
  int64_t ticket = 0;
  if (int rc = po_prefill_submit(e, tokens, n, n_cached, allowed, n_allowed, pool_block_ids, n_blocks, &ticket,
                                 stream))
    return rc;
  return po_prefill_wait(e, ticket, out_logits, out_probs, out_argmax, nullptr);
}

int po_prefill_device(po_engine* e, const uint32_t* d_tokens, int32_t n, int32_t n_cached, const int32_t* d_allowed,
                      int32_t n_allowed, const int32_t* pool_block_ids, int32_t n_blocks, float* d_logits,
                      float* d_probs, int32_t* d_argmax, void* stream) {
  if (!e || !d_tokens || !d_allowed || !d_logits || !d_probs || !d_argmax)
    return set_error(PO_ERR_ARG, "po_prefill_device: null argument");
  cudaSetDevice(e->device);
  int n_admit = 0;
  const int n_c = stage_request(e, n, n_cached, n_allowed, pool_block_ids, n_blocks, &n_admit);
  if (n_c < 0) return n_c;
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : e->stream;
  e->ring_ticket[e->cur_ring] = 0;
  const int rc = forward(e, d_tokens + n_c, n, n_c, n_admit, d_allowed, n_allowed, d_logits, d_probs, d_argmax, s);
  release_ring(e, s);
  return rc;
}

int po_engine_stream(po_engine* e, void** stream) {
  if (!e || !stream) return set_error(PO_ERR_ARG, "po_engine_stream: null argument");
  *stream = e->stream;
  return PO_OK;
}

int po_last_launches(po_engine* e, int32_t* n) {
  if (!e || !n) return set_error(PO_ERR_ARG, "po_last_launches: null argument");
  *n = e->last_launches;
  return PO_OK;
}

int po_profile_begin(po_engine* e) {
  if (!e) return set_error(PO_ERR_ARG, "po_profile_begin: null engine");
  e->profiling = true;
  e->prof_used = 0;
  return PO_OK;
}

int po_profile_end(po_engine* e, float* ms_per_class, int32_t* launches_per_class, int32_t n_classes) {
  if (!e || !ms_per_class || !launches_per_class) return set_error(PO_ERR_ARG, "po_profile_end: null argument");
  cudaSetDevice(e->device);
  for (int i = 0; i < n_classes; ++i) {
    ms_per_class[i] = 0.f;
    launches_per_class[i] = 0;
  }
  for (int i = 0; i < e->prof_used; ++i) {
    if (cudaEventSynchronize(e->prof_events[i].second) != cudaSuccess)
      return set_error(PO_ERR_CUDA, "po_profile_end: event sync failed");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e->prof_events[i].first, e->prof_events[i].second);
    const int cls = e->prof_class[i];
    if (cls < n_classes) {
      ms_per_class[cls] += ms;
      launches_per_class[cls] += 1;
    }
  }
  e->profiling = false;
  e->prof_used = 0;
  return PO_OK;
}

}  // extern "C"
