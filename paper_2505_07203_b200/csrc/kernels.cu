// Memory-bound kernels of the PrefillOnly forward: embedding gather, RMSNorm, prefix-pool KV
// gather (A/B mode only), allowed-row LM head; plus the counter-based on-device weight init.
#include "kernels.cuh"
#include <cfloat>

namespace po {

namespace {
constexpr uint64_t K_SEED = 0x9E3779B97F4A7C15ull;
constexpr uint64_t K_TID = 0xD1B54A32D192ED03ull;

__device__ __forceinline__ float unit_uniform(uint64_t seed, uint32_t tid, uint64_t idx) {
  const uint64_t z = splitmix64(seed * K_SEED + static_cast<uint64_t>(tid) * K_TID + idx);
  const float u = static_cast<float>(z >> 40) * (1.0f / 16777216.0f);  // 24-bit grid, exact in fp32
  return __fmul_rn(__fsub_rn(__fmul_rn(2.0f, u), 1.0f), 1.7320508f);
}

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  float t = (l < nw) ? red[l] : 0.f;
#pragma unroll
  for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  return t;
}
}  // namespace

__global__ void init_bf16_kernel(__nv_bfloat16* dst, long long rows, long long cols, uint64_t seed, uint32_t tid,
                                 uint32_t tid2, float scale, int mode) {
  const long long total = rows * cols;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    uint32_t t = tid;
    long long idx = i;
    if (mode == INIT_GATE_UP) {
      const long long r = i / cols, c = i - r * cols;
      const long long grp = r >> 5, w = r & 31;
      t = (w < 16) ? tid : tid2;
      idx = (grp * 16 + (w & 15)) * cols + c;
    }
    dst[i] = __float2bfloat16_rn(__fmul_rn(unit_uniform(seed, t, idx), scale));
  }
}

__global__ void init_norm_kernel(float* dst, long long n, uint64_t seed, uint32_t tid) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float g = __fadd_rn(1.0f, __fmul_rn(0.05f, unit_uniform(seed, tid, i)));
    dst[i] = __bfloat162float(__float2bfloat16_rn(g));
  }
}

__global__ void init_bias_kernel(float* dst, long long n, uint64_t seed, uint32_t tid) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = __bfloat162float(__float2bfloat16_rn(__fmul_rn(0.1f, unit_uniform(seed, tid, i))));
}
void launch_init_bias(float* dst, long long n, uint64_t seed, uint32_t tid, cudaStream_t s) {
  init_bias_kernel<<<64, 256, 0, s>>>(dst, n, seed, tid);
}

void launch_init_bf16(__nv_bfloat16* dst, long long rows, long long cols, uint64_t seed, uint32_t tid, uint32_t tid2,
                      float scale, int mode, cudaStream_t s) {
  init_bf16_kernel<<<148 * 8, 256, 0, s>>>(dst, rows, cols, seed, tid, tid2, scale, mode);
}
void launch_init_norm(float* dst, long long n, uint64_t seed, uint32_t tid, cudaStream_t s) {
  init_norm_kernel<<<64, 256, 0, s>>>(dst, n, seed, tid);
}

// ------------------------------------------------------------------ embedding (+ first folded-RMSNorm input)
// one CTA (8 warps) per row; warp w handles 128-column segments w, w + 8, ... (32 lanes x 4 columns)
__global__ void __launch_bounds__(256) embed_norm_kernel(const uint32_t* __restrict__ tokens,
                                                         const __nv_bfloat16* __restrict__ embed, int vocab,
                                                         int hidden, const float* __restrict__ gamma,
                                                         float* __restrict__ resid, __nv_bfloat16* __restrict__ xg,
                                                         float* __restrict__ ss) {
  pdl_wait();
  pdl_trigger();
  const long long r = blockIdx.x;
  const uint32_t tok = tokens[r] % static_cast<uint32_t>(vocab);
  const int nseg = hidden / 128;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int seg = warp; seg < nseg; seg += 8) {
    const int col = seg * 128 + lane * 4;
    const uint2 raw = *reinterpret_cast<const uint2*>(embed + (long long)tok * hidden + col);
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&raw);
    const float2 f0 = __bfloat1622float2(b[0]), f1 = __bfloat1622float2(b[1]);
    *reinterpret_cast<float4*>(resid + r * hidden + col) = make_float4(f0.x, f0.y, f1.x, f1.y);
    const float4 g = *reinterpret_cast<const float4*>(gamma + col);
    *reinterpret_cast<uint2*>(xg + r * hidden + col) =
        make_uint2(pack_bf16(f0.x * g.x, f0.y * g.y), pack_bf16(f1.x * g.z, f1.y * g.w));
    float sq = f0.x * f0.x + f0.y * f0.y + f1.x * f1.x + f1.y * f1.y;
#pragma unroll
    for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if (lane == 0) ss[r * nseg + seg] = sq;
  }
}
void launch_embed_norm(const uint32_t* tokens, int n, const __nv_bfloat16* embed, int vocab, int hidden,
                       const float* gamma, float* resid, __nv_bfloat16* xg, float* ss, cudaStream_t s) {
  if (n <= 0) return;
  launch_pdl(embed_norm_kernel, dim3(n), dim3(256), 0, s, tokens, embed, vocab, hidden, gamma, resid, xg, ss);
}

// ------------------------------------------------------------------ prefix pool <-> qkv
__global__ void kv_gather_kernel(const __nv_bfloat16* __restrict__ pool, const int* __restrict__ slots, int n_rows,
                                 int layer, int num_layers, int bt, int kv_dim, __nv_bfloat16* __restrict__ qkv,
                                 long long ld, int col0) {
  pdl_wait();
  pdl_trigger();
  const int vec = kv_dim / 8;
  const long long total = (long long)n_rows * vec;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(i / vec);
    const int q = static_cast<int>(i - (long long)r * vec);
    const long long slot = slots[r / bt];
    const uint4* src = reinterpret_cast<const uint4*>(pool + ((slot * num_layers + layer) * bt + (r % bt)) * kv_dim);
    reinterpret_cast<uint4*>(qkv + r * ld + col0)[q] = src[q];
  }
}
void launch_kv_gather(const __nv_bfloat16* pool, const int* slots, int n_rows, int layer, int num_layers,
                      int block_tokens, int kv_dim, __nv_bfloat16* qkv, long long ld, int col0, cudaStream_t s) {
  if (n_rows <= 0) return;
  launch_pdl(kv_gather_kernel, dim3(148 * 8), dim3(256), 0, s, pool, slots, n_rows, layer, num_layers, block_tokens,
             kv_dim, qkv, ld, col0);
}

// ------------------------------------------------------------------ allowed-row LM head
__global__ void __launch_bounds__(1024) lm_head_kernel(const float* __restrict__ x, int hidden,
                                                       const float* __restrict__ gamma, float eps,
                                                       const __nv_bfloat16* __restrict__ w,
                                                       const int* __restrict__ allowed, int n_allowed,
                                                       float* __restrict__ logits, float* __restrict__ probs,
                                                       int* __restrict__ argmax, unsigned int* __restrict__ ticket) {
  extern __shared__ float h[];  // [hidden] normalised last-row hidden state (bf16 values)
  __shared__ float red[32];
  pdl_wait();
  pdl_trigger();
  __shared__ float bmax[32];
  __shared__ int bidx[32];
  float ss = 0.f;
  for (int k = threadIdx.x; k < hidden; k += blockDim.x) ss += x[k] * x[k];
  ss = block_sum(ss, red);
  const float inv = rsqrtf(ss / hidden + eps);
  for (int k = threadIdx.x; k < hidden; k += blockDim.x)
    h[k] = __bfloat162float(__float2bfloat16_rn(x[k] * inv * gamma[k]));
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int a = blockIdx.x * nw + warp; a < n_allowed; a += gridDim.x * nw) {
    const uint4* row = reinterpret_cast<const uint4*>(w + (long long)allowed[a] * hidden);
    float acc = 0.f;
    for (int q = lane; q < hidden / 8; q += 32) {
      const uint4 v = row[q];
      const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(b[e]);
        acc += f.x * h[q * 8 + 2 * e] + f.y * h[q * 8 + 2 * e + 1];
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) logits[a] = acc;
  }
  if (gridDim.x > 1) {
    // several CTAs share the rows (long allowed lists): the last one to finish runs the softmax / argmax
    __shared__ unsigned int last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (threadIdx.x == 0) *ticket = 0;  // ready for the next launch (stream-ordered)
  }
  __threadfence_block();
  __syncthreads();
  // argmax (first index among maxima) and softmax over the allowed rows
  float m = -FLT_MAX;
  int mi = 0x7fffffff;
  for (int a = threadIdx.x; a < n_allowed; a += blockDim.x) {
    const float v = __ldcg(logits + a);  // other CTAs' rows: read at L2 (their fence + ticket ordered the stores)
    if (v > m || (v == m && a < mi)) { m = v; mi = a; }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, m, o);
    const int oi = __shfl_xor_sync(0xffffffffu, mi, o);
    if (om > m || (om == m && oi < mi)) { m = om; mi = oi; }
  }
  if (lane == 0) { bmax[warp] = m; bidx[warp] = mi; }
  __syncthreads();
  if (warp == 0) {
    m = (lane < nw) ? bmax[lane] : -FLT_MAX;
    mi = (lane < nw) ? bidx[lane] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, m, o);
      const int oi = __shfl_xor_sync(0xffffffffu, mi, o);
      if (om > m || (om == m && oi < mi)) { m = om; mi = oi; }
    }
    if (lane == 0) { bmax[0] = m; bidx[0] = mi; }
  }
  __syncthreads();
  const float gm = bmax[0];
  float se = 0.f;
  for (int a = threadIdx.x; a < n_allowed; a += blockDim.x) se += expf(__ldcg(logits + a) - gm);
  se = block_sum(se, red);
  for (int a = threadIdx.x; a < n_allowed; a += blockDim.x) probs[a] = expf(__ldcg(logits + a) - gm) / se;
  if (threadIdx.x == 0) *argmax = bidx[0];
}
// One CTA (32 warps, one allowed row each at a time) up to 256 rows: Yes/No lists are latency-bound and a single CTA
// avoids the cross-CTA hand-off. Longer lists spread the rows over up to one CTA per SM (each streams its rows'
// 8 KB at its own share of HBM), and the last CTA to finish runs the softmax / argmax; logits and probabilities are
// the same as the single-CTA kernel's (same per-row reduction, same final CTA code).
void launch_lm_head(const float* resid_row, int hidden, const float* gamma, float eps, const __nv_bfloat16* w,
                    const int* allowed, int n_allowed, float* logits, float* probs, int* argmax, unsigned int* ticket,
                    cudaStream_t s) {
  int ctas = 1;
  if (ticket && n_allowed > 256) {
    ctas = (n_allowed + 31) / 32;
    if (ctas > 148) ctas = 148;
  }
  launch_pdl(lm_head_kernel, dim3(ctas), dim3(1024), hidden * sizeof(float), s, resid_row, hidden, gamma, eps, w,
             allowed, n_allowed, logits, probs, argmax, ticket);
}

}  // namespace po
