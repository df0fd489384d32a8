// Swap-AB pair GEMM for short launches (M <= 256 rows: prefix-hit suffixes, short requests, the last layer's final row).
//
// D[M,N] = X[M,K] . W[N,K]^T with the WEIGHT as the MMA's M operand and the M activation rows as its N operand:
// tcgen05.mma.cta_group::2 M256 x N(NP) x K16, NP = M rounded up to 16. The row-major pair kernel pads M to its 256-row
// tile, so at M = 160 its tensor pipe does 1.6x the useful work per weight byte and a weight stream at HBM rate needs
// more MMA throughput than the SMs have (profiles/r1_hit_ncu_summary.json); here the MMA does exactly NP/M of it.
//
// CTA pair layout (cluster of 2, 256 threads per CTA, persistent over (weight tile, k split) units):
//   warp 0      TMA producer: per k-block its CTA's 128 weight rows (16 KB) + NP/2 activation rows
//   warp 1      MMA issuer (leader CTA): M256 NP K16 x 4 per k-block into a TMEM accumulator (double buffered)
//   warp 2      TMEM allocator
//   warps 4..7  epilogue: TMEM lane = one output column, TMEM columns = the M rows; each warp stores 32 consecutive
//               output columns of one row per instruction (coalesced), either the fused epilogue (BF16, F32,
//               SiLU.mul) or, for split-K units, the fp32 partial that splitk_reduce_kernel sums in split order.
#include "gemm.cuh"
#include "gemm_epi.cuh"
#include <cstdlib>
#include <cstring>

namespace po {

#ifdef SWAP_TRACE
// globaltimer stamps per CTA (tools/dbg_swap_trace.py): 0 start, 1 after setup, 2 first full barrier seen by the MMA
// thread, 3 last MMA commit, 4 epilogue start (first tfull), 5 epilogue done, 6 exit, 7 last unit's epilogue start
__device__ unsigned long long g_swap_trace[296 * 16];
__device__ __forceinline__ unsigned long long gtime_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#ifndef SWAP_TRACE_N
#define SWAP_TRACE_N 0
#endif
#define STAMP(i, cond) \
  do {                 \
    if ((cond) && (SWAP_TRACE_N == 0 || (args.N == SWAP_TRACE_N && args.M > 1))) \
      g_swap_trace[blockIdx.x * 16 + (i)] = gtime_ns(); \
  } while (0)
#else
#define STAMP(i, cond) \
  do {                 \
  } while (0)
#endif

namespace {
constexpr int BK = 64;
constexpr int W_BYTES = 128 * BK * 2;  // 16 KB: this CTA's 128 weight rows of a k-block
constexpr int X_MAX = 128 * BK * 2;    // up to 128 activation rows (NP <= 256, half per CTA)
constexpr int STAGE = W_BYTES + X_MAX;
constexpr int STAGES = 6;
constexpr int STG = 4 * 2 * 4096;      // epilogue staging: per warp two 32 x 32 fp32 boxes for TMA stores
constexpr int SMEM = STAGES * STAGE + STG + 1024 + 256 + 1024;
constexpr int NT = 256;
constexpr int ACC_STRIDE = 256;  // TMEM columns between the two accumulators
}  // namespace

template <int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT, 1)
    gemm2s_kernel(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x,
                  const __grid_constant__ CUtensorMap map_st, const GemmArgs args, int np) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint8_t* sW = smem;
  uint8_t* sX = smem + STAGES * W_BYTES;
  uint8_t* stg = smem + STAGES * STAGE;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE + STG);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  float* s_inv = reinterpret_cast<float*>(smem + STAGES * STAGE + STG + 256);  // 1/rms per activation row (<= 256)

  const int warp = warp_id();
  const int lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  const int npairs = gridDim.x >> 1;
  const int num_n = args.N / 256;
  const int ksp = args.k_splits > 1 ? args.k_splits : 1;
  const int num_units = num_n * ksp;
  const int nk_total = args.K / BK;
  const int kbps = ksp > 1 ? args.kb_per_split : nk_total;
  const int xh = np / 2;  // activation rows per CTA
  const uint32_t x_bytes = (uint32_t)xh * BK * 2;
  STAMP(0, threadIdx.x == 0);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_w);
    tma_prefetch_desc(&map_x);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 2);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  STAMP(1, threadIdx.x == 0);
  // weights are constant: the producer streams its first STAGES weight k-blocks before waiting for the kernel that
  // writes the activations
  if (warp != 0) pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t full0 = mapa_shared(smem_u32(full_bar), 0);
      int s = 0;
      uint32_t ph = 0;
      int pend_s[STAGES], pend_kb[STAGES];
      int npend = 0;
      bool open = false;
      const int xrow = args.a_row0 + (int)rank * xh;
      auto flush = [&]() {
        pdl_wait();
        open = true;
        for (int i = 0; i < npend; ++i)
          tma_load_2d_pair(sX + pend_s[i] * X_MAX, &map_x, full0 + pend_s[i] * 8, pend_kb[i] * BK, xrow);
        npend = 0;
      };
      for (int u = pair; u < num_units; u += npairs) {
        const int nb = u / ksp;
        const int kb0 = (u % ksp) * kbps;
        const int nk = min(nk_total, kb0 + kbps) - kb0;
        for (int k = 0; k < nk; ++k) {
          const int kb = kb0 + k;
          mbar_wait(&empty_bar[s], ph ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&full_bar[s], 2 * (W_BYTES + x_bytes));
          const uint32_t fb = full0 + s * 8;
          tma_load_2d_pair(sW + s * W_BYTES, &map_w, fb, kb * BK, nb * 256 + (int)rank * 128);
          if (open) {
            tma_load_2d_pair(sX + s * X_MAX, &map_x, fb, kb * BK, xrow);
          } else {
            pend_s[npend] = s;
            pend_kb[npend] = kb;
            if (++npend == STAGES) flush();
          }
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
      }
      if (!open) flush();
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      const uint32_t idesc = idesc_bf16_f32(256, (uint32_t)np);
      int s = 0;
      uint32_t ph = 0;
      int it = 0;
      for (int u = pair; u < num_units; u += npairs, ++it) {
        const int acc = it & 1;
        const uint32_t acc_ph = (it >> 1) & 1;
        mbar_wait(&tempty_bar[acc], acc_ph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * ACC_STRIDE;
        const int kb0 = (u % ksp) * kbps;
        const int nk = min(nk_total, kb0 + kbps) - kb0;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full_bar[s], ph);
          tc_fence_after();
          STAMP(2, it == 0 && kb == 0);
          const uint64_t adesc = sdesc_kmajor_sw128(smem_u32(sW + s * W_BYTES));
          const uint64_t bdesc = sdesc_kmajor_sw128(smem_u32(sX + s * X_MAX));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) mma_bf16_ss_pair(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
          mma_commit_pair(&empty_bar[s], 0x3);
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
        mma_commit_pair(&tfull_bar[acc], 0x3);
        STAMP(3, true);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int wq = warp & 3;
    const int et = threadIdx.x - 128;
    const uint32_t tempty0 = mapa_shared(smem_u32(tempty_bar), 0);
    if (EPI == EPI_SILU_MUL && ksp == 1) {  // 1/rms of every activation row, once (the rows are the same for all units)
      for (int r = et; r < args.M; r += 128) s_inv[r] = args.ss_in ? row_inv_rms(args, r) : 1.0f;
      named_bar_sync(1, 128);
    }
    int it = 0;
    int nst = 0;  // TMA-store boxes issued by this warp (staging buffer nst & 1)
    for (int u = pair; u < num_units; u += npairs, ++it) {
      const int nb = u / ksp;
      const int acc = it & 1;
      const uint32_t acc_ph = (it >> 1) & 1;
      mbar_wait(&tfull_bar[acc], acc_ph);
      tc_fence_after();
      STAMP(4, et == 0 && it == 0);
      STAMP(7, et == 0);
      const int col = nb * 256 + (int)rank * 128 + wq * 32 + lane;  // this thread's output column
      const uint32_t taddr = tmem_base + ((uint32_t)(wq * 32) << 16) + acc * ACC_STRIDE;
#pragma unroll 1
      for (int c0 = 0; c0 < args.M; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(taddr + c0, r);
        tmem_ld_wait();
        // Every mode stages this warp's 32 activation rows x 32 output columns in shared memory (row-major, one row
        // per activation row) and writes the box with one TMA store; rows >= M are clipped by the map's bounds.
        //   split-K: fp32 partial [split][row][col] (map_st over the workspace); F32 / BF16: the output;
        //   SiLU.mul: 16 bf16 output columns per warp
        uint8_t* wb = stg + (wq * 2 + (nst & 1)) * 4096;
        STAMP(8 + 4 * (c0 / 32), et == 0 && u + npairs >= num_units && c0 < 64);
        if (lane == 0) bulk_wait_read<1>();  // the store that last read this buffer (two boxes ago) is done
        __syncwarp();
        STAMP(9 + 4 * (c0 / 32), et == 0 && u + npairs >= num_units && c0 < 64);
        int sc0 = col - lane;
        if (ksp > 1 || EPI == EPI_F32) {
          float* t = reinterpret_cast<float*>(wb);
#pragma unroll
          for (int j = 0; j < 32; ++j) t[j * 32 + lane] = __uint_as_float(r[j]);
        } else if constexpr (EPI == EPI_BF16) {
          __nv_bfloat16* t = reinterpret_cast<__nv_bfloat16*>(wb);
#pragma unroll
          for (int j = 0; j < 32; ++j) t[j * 32 + lane] = __float2bfloat16_rn(__uint_as_float(r[j]));
        } else if constexpr (EPI == EPI_SILU_MUL) {
          // weight rows come in 16-row groups [gate 16 | up 16]: lanes 0..15 hold gate columns, 16..31 the matching
          // up columns; output column (col / 32) * 16 + col % 32 (the row-major epilogue's interleave)
          // Two activation rows per step with every lane busy: lanes 0..15 finish row j (own gate, partner's up),
          // lanes 16..31 row j + 1 (partner's gate, own up); one shuffle per pair of rows, no divergence.
          __nv_bfloat16* t = reinterpret_cast<__nv_bfloat16*>(wb);
          const bool hi = lane >= 16;
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const float mine = __uint_as_float(hi ? r[j] : r[j + 1]);
            const float other = __shfl_xor_sync(0xffffffffu, mine, 16);
            const float g = hi ? other : __uint_as_float(r[j]);
            const float up = hi ? __uint_as_float(r[j + 1]) : other;
            const int row = j + (hi ? 1 : 0);
            const float sc = s_inv[min(c0 + row, 255)];
            t[row * 16 + (lane & 15)] = __float2bfloat16_rn(silu_f(sc * g) * (sc * up));
          }
          sc0 /= 2;
        }
        STAMP(10 + 4 * (c0 / 32), et == 0 && u + npairs >= num_units && c0 < 64);
        fence_proxy_async_smem();
        __syncwarp();
        STAMP(11 + 4 * (c0 / 32), et == 0 && u + npairs >= num_units && c0 < 64);
#ifndef SWAP_NO_TMA_STORE
        if (lane == 0) {
          tma_store_3d(&map_st, wb, sc0, c0, ksp > 1 ? u % ksp : 0);
          bulk_commit();
        }
#endif
        STAMP(14, et == 0 && u + npairs >= num_units && c0 == 0);
        ++nst;
      }
      tc_fence_before();
      named_bar_sync(1, 128);
      if (threadIdx.x == 128) mbar_arrive_cluster(tempty0 + acc * 8);
      STAMP(5, et == 0);
    }
    if (lane == 0) bulk_wait_all();  // partials written (and the staging buffers read) before the CTA exits
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 512);
  }
  STAMP(6, threadIdx.x == 0);
}

// The swap-AB kernel covers a launch when every unit ends in a split-K partial (reduce kernel applies the epilogue)
// or the epilogue is one of the transposed ones above.
// PO_SWAP_AB=0 keeps the row-major kernels for short launches (A/B runs)
bool gemm_swap_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* v = getenv("PO_SWAP_AB");
    on = (v && v[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

bool gemm_swap_supported(int epi, int M, int N, int K, bool split) {
  if (M < 1 || M > 256 || N % 256 || K % BK) return false;
  return split || epi == EPI_BF16 || epi == EPI_F32 || epi == EPI_SILU_MUL;
}

int splitk_reduce_launch(int epi, const GemmArgs& args, cudaStream_t stream);

// Returns 0, a negative error, or 1 when this launch is not covered (the caller runs the row-major kernels).
// map_w: the weight with 128-row boxes (the pair kernel's map_b2). x / ldx: the activation buffer (rows a_row0 ..
// a_row0 + M - 1 are read; the map is bounded there, so the rounding rows of NP are zero-filled by TMA).
#ifdef SWAP_NO_PDL
#define PO_SWAP_LAUNCH(k, g, b, sm, st, ...) k<<<g, b, sm, st>>>(__VA_ARGS__)
#else
#define PO_SWAP_LAUNCH(k, g, b, sm, st, ...) launch_pdl(k, g, b, sm, st, __VA_ARGS__)
#endif
int gemm_launch_swap(const CUtensorMap& map_w, const void* x, long long ldx, int epi, const GemmArgs& in,
                     cudaStream_t stream) {
  GemmArgs args = in;
  args.k_splits = 1;
  const int np = (args.M + 15) / 16 * 16;
  const int tiles = args.N / 256;
  const int pairs = num_sms() / 2;
  const int nk = args.K / BK;
  if (args.split_ws && tiles * 2 <= pairs && nk >= 16) {
    int s = pairs / tiles;
    s = s < nk / 8 ? s : nk / 8;
    if (s > 1) {
      args.kb_per_split = (nk + s - 1) / s;
      args.k_splits = (nk + args.kb_per_split - 1) / args.kb_per_split;
      if ((size_t)args.k_splits * args.M * args.N * sizeof(float) > args.split_ws_bytes) args.k_splits = 1;
    }
  }
  if (!gemm_swap_supported(epi, args.M, args.N, args.K, args.k_splits > 1)) return 1;  // not handled: caller falls back
  CUtensorMap map_x, map_st;
  if (make_tmap_2d_bf16(&map_x, x, args.K, (uint64_t)args.a_row0 + args.M, ldx * 2, BK, np / 2)) return -2;
  // the epilogue's TMA-store map: split-K partials [split][M][N] fp32, or the output [M][N] (row stride ldo)
  int mrc;
  if (args.k_splits > 1)
    mrc = make_tmap_store_3d(&map_st, args.split_ws, true, args.N, args.M, args.k_splits, (uint64_t)args.N * 4,
                             (uint64_t)args.N * args.M * 4, 32, 32);
  else if (epi == EPI_F32)
    mrc = make_tmap_store_3d(&map_st, args.out, true, args.N, args.M, 1, (uint64_t)args.ldo * 4,
                             (uint64_t)args.ldo * 4 * args.M, 32, 32);
  else if (epi == EPI_BF16)
    mrc = make_tmap_store_3d(&map_st, args.out, false, args.N, args.M, 1, (uint64_t)args.ldo * 2,
                             (uint64_t)args.ldo * 2 * args.M, 32, 32);
  else
    mrc = make_tmap_store_3d(&map_st, args.out, false, args.N / 2, args.M, 1, (uint64_t)args.ldo * 2,
                             (uint64_t)args.ldo * 2 * args.M, 16, 32);
  if (mrc) return 1;  // output not TMA-addressable (alignment): row-major kernels
  const int units = tiles * args.k_splits;
  const int np_pairs = units < pairs ? units : pairs;
  switch (epi) {
#define PO_SWAP_CASE(E)                                                                                  \
  case E:                                                                                                \
    ensure_smem_attr<gemm2s_kernel<E>>(SMEM);                                                            \
    PO_SWAP_LAUNCH(gemm2s_kernel<E>, dim3(2 * np_pairs), dim3(NT), SMEM, stream, map_w, map_x, map_st, args, np); \
    break;
    PO_SWAP_CASE(EPI_BF16)
    PO_SWAP_CASE(EPI_F32)
    PO_SWAP_CASE(EPI_SILU_MUL)
    PO_SWAP_CASE(EPI_RESID_F32)
    PO_SWAP_CASE(EPI_QKV_ROPE)
#undef PO_SWAP_CASE
    default: return -3;
  }
  if (args.k_splits > 1) return splitk_reduce_launch(epi, args, stream);
  return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

}  // namespace po

#ifdef SWAP_TRACE
extern "C" int po_debug_swap_trace(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, po::g_swap_trace, sizeof(unsigned long long) * 296 * 16) == cudaSuccess ? 0 : -1;
}
#endif
