// Persistent weight-streaming layer kernel for short requests (prefix hits: M <= 256 miss rows).
//
// A prefix hit's layer GEMMs are weight streams (M = 160 rows against 25-117 M-parameter matrices), and as separate
// launches each loses a quarter to a third of its span to launch ramp, tail and a split-K reduce launch
// (profiles/r1_hit_launches_summary.md). This kernel keeps one CTA pair per SM pair resident and runs up to
// STREAM_MAX_PHASES dependent GEMMs of a layer (O-proj -> gate/up -> down -> next layer's QKV) as phases:
//   * work split: each phase's (weight tile, k-block) space is cut into equal contiguous ranges, one per CTA pair
//     (stream-K), so every pair streams the same number of weight bytes in every phase;
//   * fix-up: a tile that lies inside one pair's range gets its fused epilogue straight from TMEM. A tile cut across
//     pairs is cut at most at its ends of each pair's range, so its segments are the last unit of one pair and the
//     first units of the next ones: each segment dumps its fp32 partial and raises a flag, and once a pair has dumped
//     all its units the tile's 2 x nseg CTAs sum all segments (in segment order) for interleaved shares of the rows
//     and run the fused epilogue. No reduce launch exists, the work is spread over the tile's owners, and the
//     summation order is fixed;
//   * phases are separated by a grid barrier (one counter, monotonic across launches); before waiting on it the TMA
//     producer already streams the next phase's first weight k-blocks into the free stages (weights do not depend on
//     the previous phase), so the DRAM pipe stays busy across the barrier.
// The epilogues are the per-GEMM kernels' (gemm_epi.cuh): RoPE + admission, SiLU.mul, residual + next-norm input.
#pragma once
#include "gemm.cuh"

namespace po {

constexpr int STREAM_MAX_PHASES = 4;

struct alignas(64) StreamPhase {
  CUtensorMap a;  // activation [rows, K] bf16, 128-row boxes, bounded at g.a_row0 + g.M rows
  CUtensorMap b;  // weight [N, K] bf16, 128-row boxes (the pair kernel's map2_*)
  GemmArgs g;     // M (<= 256), N, K, a_row0 and the epilogue fields
  int epi;        // EPI_RESID_F32 / EPI_SILU_MUL / EPI_QKV_ROPE / EPI_BF16
  int slots_per_tile;  // partial slots per weight tile (max segments - 1), set by stream_launch
};

struct StreamArgs {
  StreamPhase ph[STREAM_MAX_PHASES];
  int nph;
  float* ws;                  // partial tiles [tile][slot][M][256] fp32
  size_t ws_bytes;
  uint32_t* flags;            // per (slot, CTA rank): tag of the phase that last wrote it
  size_t n_flags;
  unsigned long long* bar;    // grid-barrier counter (monotonic)
  unsigned long long bar_base;  // its value when this launch starts
  uint32_t tag;               // launch tag; a phase's flag value is tag * 8 + phase
};

// Equal contiguous k-block ranges: pair q owns [start(q), start(q + 1)) of the phase's W = tiles * k-blocks.
__host__ __device__ inline int stream_pair_start(long long W, int P, int q) { return (int)((long long)q * W / P); }
// The pair whose range holds k-block kb (the largest q with start(q) <= kb; never an empty range).
__host__ __device__ inline int stream_owner(long long W, int P, int kb) {
  int q = (int)(((long long)kb * P) / W);
  while (q + 1 < P && stream_pair_start(W, P, q + 1) <= kb) ++q;
  while (q > 0 && stream_pair_start(W, P, q) > kb) --q;
  return q;
}

// Pairs the kernel runs on (one CTA pair per two SMs) and the grid-barrier arrivals one launch adds.
int stream_pairs();
// Workspace bytes / flag count a phase of this shape needs at M rows.
size_t stream_ws_bytes(int M, int N, int K);
size_t stream_flag_count(int N, int K);
// Fill slots_per_tile, check the workspace, launch (PDL). Returns 0, -3 (shape / workspace) or -4 (launch).
// On success the caller advances bar_base by nph * 2 * stream_pairs() and the tag by one.
int stream_launch(StreamArgs& args, cudaStream_t stream);

}  // namespace po
