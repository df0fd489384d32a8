// Fused per-layer MLP launch (mlp.cu): gate/up + SiLU.mul and down + residual tiles of all row pieces in one
// persistent grid, the [piece, d_ff] intermediate in an L2-pinned two-buffer ring.
#pragma once
#include "gemm.cuh"

namespace po {

struct MlpArgs {
  GemmArgs gu;      // gate/up: N = 2 d_ff, K = hidden, out = the act ring (2 x piece rows, ld d_ff), ss_in (rows 0..)
  GemmArgs dn;      // down: N = hidden, K = d_ff, resid / xg_out / ss_out / g_next (rows 0..)
  int rows;         // MLP rows of the launch
  int piece;        // rows per piece (the ring holds two)
  int npieces, max_rbs, n_gu, n_d, total, npairs;  // filled by mlp_launch
  int* cnt;         // completion counters [npieces][max_rbs] (gate/up) + [npieces] (down), zero between launches
  unsigned int* ticket;
  int* next;        // tile fetch counter (zero between launches)
};

bool mlp_fused_enabled();
size_t mlp_counter_ints(long long max_rows, int piece);
// map_xg / map_act: 128-row activation boxes; map_wgu / map_wd: 128-row weight boxes (the pair kernel's map_b2).
int mlp_launch(const CUtensorMap& map_xg, const CUtensorMap& map_wgu, const CUtensorMap& map_act,
               const CUtensorMap& map_wd, const MlpArgs& a, cudaStream_t stream);

}  // namespace po
