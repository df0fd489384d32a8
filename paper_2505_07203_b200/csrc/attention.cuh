// Host interface of the attention kernels (attention.cu), shared by the engine and the C-ABI op.
#pragma once
#include <cstddef>
#include <cuda_runtime.h>

namespace po {

// Pool-direct key source of one attention launch: the prefix pool [num_blocks][num_layers][16][kv_dim] bf16 and the
// request's per-block slots; key rows [0, n_rows) are read from the pool, the rest from qkv.
struct AttnPool {
  const void* base;
  const int* slots;
  int n_rows;  // cached key rows (multiple of 16) read from the pool
  int num_blocks, num_layers, layer, kv_dim, block_tokens;
};

// Causal GQA attention over qkv[n_total, ld] (Q | K | V columns) for query rows [q_offset, n_total) into
// out[n_total - q_offset, ldo]. workspace: split-KV partials (attention_workspace_bytes), pool: optional key source.
// Returns 0, -2 (tensor map), -3 (shape) or -4 (launch).
int attention_run(const void* qkv, long long ld, int n_total, int q_offset, int hq, int hkv, void* out, long long ldo,
                  cudaStream_t stream, void* workspace, size_t workspace_bytes, const AttnPool* pool);
size_t attention_workspace_bytes(int n_total, int q_offset, int hq, int hkv);

}  // namespace po
