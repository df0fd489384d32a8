// Memory-bound kernels of the PrefillOnly forward (HBM-roofline kernels) and on-device weight init.
#pragma once
#include "sm100.cuh"

namespace po {

// Counter-based uniform in [-sqrt3, sqrt3) (unit variance); the CPU oracle reproduces it bit for bit.
__host__ __device__ inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// Weight-init modes
enum InitMode : int {
  INIT_PLAIN = 0,       // dst[i] = w(tid, i)
  INIT_GATE_UP = 1,     // dst rows interleave gate/up in 16-row groups (tid = gate id, tid2 = up id)
  INIT_NORM = 2,        // dst (fp32) = bf16(1 + 0.05 * u)
};

void launch_init_bf16(__nv_bfloat16* dst, long long rows, long long cols, uint64_t seed, uint32_t tid, uint32_t tid2,
                      float scale, int mode, cudaStream_t s);
void launch_init_norm(float* dst, long long n, uint64_t seed, uint32_t tid, cudaStream_t s);
// dst (fp32) = bf16(0.1 * u): random-init q/k/v bias
void launch_init_bias(float* dst, long long n, uint64_t seed, uint32_t tid, cudaStream_t s);

// resid[r, :] = float(embed[tokens[r] % vocab, :]); xg[r, :] = bf16(resid . gamma); ss[r][seg] = sum of resid^2 over
// 128-column segment seg (the first layer's folded RMSNorm input, see GemmArgs)
void launch_embed_norm(const uint32_t* tokens, int n, const __nv_bfloat16* embed, int vocab, int hidden,
                       const float* gamma, float* resid, __nv_bfloat16* xg, float* ss, cudaStream_t s);
// Prefix pool -> layer qkv buffer (only with PO_POOL_DIRECT=0; admission is stored by the QKV GEMM epilogue).
// Pool layout: [slot][layer][block_tokens][kv_dim] bf16.
void launch_kv_gather(const __nv_bfloat16* pool, const int* slots, int n_rows, int layer, int num_layers,
                      int block_tokens, int kv_dim, __nv_bfloat16* qkv, long long ld, int col0, cudaStream_t s);
// Last-row final norm + allowed-row LM head + restricted softmax + argmax.
void launch_lm_head(const float* resid_row, int hidden, const float* gamma, float eps, const __nv_bfloat16* w,
                    const int* allowed, int n_allowed, float* logits, float* probs, int* argmax, unsigned int* ticket,
                    cudaStream_t s);

}  // namespace po
