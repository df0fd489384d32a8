// tcgen05 GEMM for sm_100a. See gemm.cuh for the contract.
//
// CTA layout (256 threads, 1 CTA per SM, persistent over output tiles):
//   warp 0      TMA producer (one lane): A 128x64 + B 256x64 bf16 per stage, 128B swizzle
//   warp 1      MMA issuer (one lane): 4 x tcgen05.mma M128 N256 K16 per stage into a TMEM accumulator
//   warp 2      TMEM allocator (512 columns = two 256-column accumulators, double buffered)
//   warps 4..7  epilogue: tcgen05.ld 32 rows x 32 columns per warp, fused op, global store
// Pipelines: smem full/empty ring (TMA <-> MMA) and TMEM full/empty pair (MMA <-> epilogue).
#include "gemm.cuh"
#include "gemm_epi.cuh"
#include "stream.cuh"
#include <cuda_fp8.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>

namespace po {

namespace {
constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 64;
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;            // 16 KB
constexpr int B_BYTES = BN * BK * 2;            // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;  // 48 KB
constexpr int NUM_THREADS = 256;
constexpr int GROUP_M = 16;                     // tile raster: 16 m-blocks share each n sweep
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
}  // namespace

__device__ __forceinline__ void tile_coords(int t, int num_m, int num_n, int& m_blk, int& n_blk, int gm = GROUP_M) {
  const int per_group = gm * num_n;
  const int g = t / per_group;
  const int first_m = g * gm;
  const int gsz = min(num_m - first_m, gm);
  const int local = t - g * per_group;
  m_blk = first_m + local % gsz;
  n_blk = local / gsz;
}

template <int EPI>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                const GemmArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = warp_id();
  const int lane = lane_id();
  const int num_m = (args.M + BM - 1) / BM;
  const int num_n = args.N / BN;
  const int ksp = args.k_splits > 1 ? args.k_splits : 1;
  const int num_tiles = num_m * num_n * ksp;
  const int nk_total = args.K / BK;
  const int kbps = ksp > 1 ? args.kb_per_split : nk_total;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 128);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();     // the previous kernel's outputs (our A operand / residual) are complete from here on
  pdl_trigger();  // let the next kernel of the forward start its prologue on SMs we free

  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int mb, nb;
        tile_coords(t / ksp, num_m, num_n, mb, nb, args.group_m > 0 ? args.group_m : GROUP_M);
        const int kb0 = (t % ksp) * kbps;
        const int nk = min(nk_total, kb0 + kbps) - kb0;
        for (int k = 0; k < nk; ++k) {
          const int kb = kb0 + k;
          mbar_wait(&empty_bar[s], ph ^ 1);
          mbar_arrive_expect_tx(&full_bar[s], STAGE_BYTES);
          tma_load_2d(sA + s * A_BYTES, &map_a, &full_bar[s], kb * BK, args.a_row0 + mb * BM);
          tma_load_2d(sB + s * B_BYTES, &map_b, &full_bar[s], kb * BK, nb * BN);
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(BM, BN);
      int s = 0;
      uint32_t ph = 0;
      int it = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
        const int acc = it & 1;
        const uint32_t acc_ph = (it >> 1) & 1;
        mbar_wait(&tempty_bar[acc], acc_ph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        const int kb0 = (t % ksp) * kbps;
        const int nk = min(nk_total, kb0 + kbps) - kb0;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full_bar[s], ph);
          tc_fence_after();
          const uint64_t adesc = sdesc_kmajor_sw128(smem_u32(sA + s * A_BYTES));
          const uint64_t bdesc = sdesc_kmajor_sw128(smem_u32(sB + s * B_BYTES));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // advance 16 bf16 = 32 bytes along K inside the swizzle atom (descriptor units of 16 B)
            mma_bf16_ss(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
          }
          mma_commit(&empty_bar[s]);
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
        mma_commit(&tfull_bar[acc]);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int wq = warp & 3;  // TMEM lane quadrant this warp may access
    int it = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
      int mb, nb;
      tile_coords(t / ksp, num_m, num_n, mb, nb, args.group_m > 0 ? args.group_m : GROUP_M);
      const int acc = it & 1;
      const uint32_t acc_ph = (it >> 1) & 1;
      mbar_wait(&tfull_bar[acc], acc_ph);
      tc_fence_after();
      const int row = mb * BM + wq * 32 + lane;
      const uint32_t taddr = tmem_base + ((uint32_t)(wq * 32) << 16) + acc * BN;
      epilogue_tile<EPI>(args, taddr, row, nb, ksp, t);
      tc_fence_before();
      mbar_arrive(&tempty_bar[acc]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}


// ------------------------------------------------------------------ 2-CTA (cta_group::2) variant
// A CTA pair computes a 256 x 256 tile: each CTA loads its own 128 rows of A and 128 of the 256 B rows (the
// pair's MMA reads both CTAs' shared memory), so per-CTA B traffic halves vs the 1-CTA 128 x 256 tile. The
// leader CTA (rank 0) issues tcgen05.mma.cta_group::2 (M256 N256 K16); both CTAs' TMA loads complete on the
// leader's full barrier; MMA commits multicast to both CTAs' empty / tmem-full barriers; each CTA drains its
// own 128 accumulator rows and reports to the leader's tmem-empty barrier.
namespace {
constexpr int HALF_BYTES = 128 * BK * 2;             // 16 KB: 128 rows x 64 bf16 (A half per CTA)
template <int BNT>
struct Pair {
  static constexpr int B_BYTES = (BNT / 2) * BK * 2;  // B half per CTA
  static constexpr int STAGE = HALF_BYTES + B_BYTES;
  static constexpr int STAGES = 192 * 1024 / STAGE;  // 6 (BNT 256) or 8 (BNT 128)
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
};
}  // namespace

// F8: E4M3 operands (kind::f8f6f4); a k-block is still one 128-byte row per operand row (128 elements instead of 64)
// EW: epilogue warps per TMEM lane quadrant (1: warps 4..7 drain whole tiles; 2: warps 4..11, each pair of warps of a
// quadrant splits the tile's columns in 128-column halves). EW = 2 measured slower on the 20k step (QKV 24.4 -> 29.8
// ms, O-proj 21.8 -> 21.3 ms: the O-proj is not bound by its epilogue warps' issue rate), so every variant uses 1.
template <int EW>
constexpr int pair_threads() { return 128 + 128 * EW; }
template <bool F8, int BNT>
constexpr int pair_ew() { return 1; }

// RT (EPI_RESID_F32, bf16, 256-wide tiles): the residual read-modify-write goes through shared memory by TMA. Per
// epilogue warp and 32-column chunk, a [32 rows x 32 fp32] box of the residual is loaded one chunk ahead (128-byte
// swizzle: float4 q of row r at q ^ (r & 7), conflict-free for the thread-per-row access), updated in place, and
// stored back with the bf16 folded-norm input box by TMA, instead of per-thread 128-byte row segments (32 L2 lines
// per warp instruction, in both directions). One pipeline stage fewer pays for the 48 KB of staging.
constexpr int RT_WARP_BYTES = 2 * 4096 + 2 * 2048;  // per epilogue warp: two residual boxes + two xg boxes
template <int EPI, int BNT, bool F8>
constexpr bool pair_rt() { return EPI == EPI_RESID_F32 && BNT == 256; }
template <int EPI, int BNT, bool F8>
constexpr int pair_stages() { return pair_rt<EPI, BNT, F8>() ? Pair<BNT>::STAGES - 1 : Pair<BNT>::STAGES; }
template <int EPI, int BNT, bool F8>
constexpr int pair_smem() {
  return pair_stages<EPI, BNT, F8>() * Pair<BNT>::STAGE + (pair_rt<EPI, BNT, F8>() ? 4 * RT_WARP_BYTES : 0) + 1024 +
         256;
}

template <int EPI, int BNT, bool F8 = false, int EW = pair_ew<F8, BNT>()>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(pair_threads<EW>(), 1)
    gemm2_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                 const __grid_constant__ CUtensorMap map_r, const __grid_constant__ CUtensorMap map_xo,
                 const GemmArgs args) {
  constexpr int KE = F8 ? 2 * BK : BK;  // k elements per k-block
  constexpr bool RT = pair_rt<EPI, BNT, F8>();
  constexpr int STAGES2 = pair_stages<EPI, BNT, F8>();
  constexpr int B_HALF = Pair<BNT>::B_BYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES2 * HALF_BYTES;
  uint8_t* rt_stg = smem + STAGES2 * Pair<BNT>::STAGE;  // RT staging (4 warps x RT_WARP_BYTES)
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(rt_stg + (RT ? 4 * RT_WARP_BYTES : 0));
  uint64_t* empty_bar = full_bar + STAGES2;
  uint64_t* tfull_bar = empty_bar + STAGES2;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* rt_bar = tempty_bar + 2;  // [4 warps][2 buffers] residual box loads (RT)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rt_bar + 8);

  const int warp = warp_id();
  const int lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  const int npairs = gridDim.x >> 1;
  const int num_m = (args.M + 2 * BM - 1) / (2 * BM);
  const int num_n = args.N / BNT;
  const int ksp = args.k_splits > 1 ? args.k_splits : 1;
  const int num_tiles = num_m * num_n * ksp;
  const int nk_total = args.K / KE;
  const int kbps = ksp > 1 ? args.kb_per_split : nk_total;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    for (int s = 0; s < STAGES2; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 2);  // one arrival per CTA of the pair (leader's copy is the one used)
    }
    if (RT)
      for (int s = 0; s < 8; ++s) mbar_init(&rt_bar[s], 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair(tmem_slot, 2 * BNT);
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // peer barriers initialised before any remote arrive / TMA completion
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // The producer streams its first STAGES2 weight k-blocks before waiting for the previous kernel (weights are
  // constant; only the activation rows depend on it), so the weight fetch overlaps the predecessor's tail.
  if (warp != 0) pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t full0 = mapa_shared(smem_u32(full_bar), 0);  // leader's full_bar[0]
      int s = 0;
      uint32_t ph = 0;
      int pend_s[STAGES2], pend_kb[STAGES2], pend_row[STAGES2];
      int npend = 0;
      bool open = false;
      auto flush = [&]() {
        pdl_wait();
        open = true;
        for (int i = 0; i < npend; ++i)
          tma_load_2d_pair(sA + pend_s[i] * HALF_BYTES, &map_a, full0 + pend_s[i] * 8, pend_kb[i] * KE, pend_row[i]);
        npend = 0;
      };
      for (int t = pair; t < num_tiles; t += npairs) {
        int mb, nb;
        tile_coords(t / ksp, num_m, num_n, mb, nb, args.group_m > 0 ? args.group_m : GROUP_M);
        const int kb0 = (t % ksp) * kbps;
        const int nk = min(nk_total, kb0 + kbps) - kb0;
        const int arow = args.a_row0 + mb * 2 * BM + rank * BM;
        for (int k = 0; k < nk; ++k) {
          const int kb = kb0 + k;
          mbar_wait(&empty_bar[s], ph ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&full_bar[s], 2 * Pair<BNT>::STAGE);
          const uint32_t fb = full0 + s * 8;
          tma_load_2d_pair(sB + s * B_HALF, &map_b, fb, kb * KE, nb * BNT + rank * (BNT / 2));
          if (open) {
            tma_load_2d_pair(sA + s * HALF_BYTES, &map_a, fb, kb * KE, arow);
          } else {
            pend_s[npend] = s;
            pend_kb[npend] = kb;
            pend_row[npend] = arow;
            if (++npend == STAGES2) flush();
          }
          if (++s == STAGES2) { s = 0; ph ^= 1; }
        }
      }
      if (!open) flush();
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = F8 ? idesc_e4m3_f32(2 * BM, BNT) : idesc_bf16_f32(2 * BM, BNT);
      int s = 0;
      uint32_t ph = 0;
      int it = 0;
      for (int t = pair; t < num_tiles; t += npairs, ++it) {
        const int acc = it & 1;
        const uint32_t acc_ph = (it >> 1) & 1;
        mbar_wait(&tempty_bar[acc], acc_ph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BNT;
        const int kb0 = (t % ksp) * kbps;
        const int nk = min(nk_total, kb0 + kbps) - kb0;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full_bar[s], ph);
          tc_fence_after();
          const uint64_t adesc = sdesc_kmajor_sw128(smem_u32(sA + s * HALF_BYTES));
          const uint64_t bdesc = sdesc_kmajor_sw128(smem_u32(sB + s * B_HALF));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {  // 4 MMAs of 32 bytes of K each (K16 bf16 or K32 e4m3)
            if constexpr (F8)
              mma_f8_ss_pair(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
            else
              mma_bf16_ss_pair(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
          }
          mma_commit_pair(&empty_bar[s], 0x3);
          if (++s == STAGES2) { s = 0; ph ^= 1; }
        }
        mma_commit_pair(&tfull_bar[acc], 0x3);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int wq = warp & 3;
    constexpr int CW = BNT / EW;  // columns per epilogue warp of a quadrant
    const int part = (warp - 4) >> 2;
    const uint32_t tempty0 = mapa_shared(smem_u32(tempty_bar), 0);
    int rt_ph[2] = {0, 0};  // RT: parity of each residual buffer's next load
    int it = 0;
    for (int t = pair; t < num_tiles; t += npairs, ++it) {
      int mb, nb;
      tile_coords(t / ksp, num_m, num_n, mb, nb, args.group_m > 0 ? args.group_m : GROUP_M);
      const int acc = it & 1;
      const uint32_t acc_ph = (it >> 1) & 1;
      mbar_wait(&tfull_bar[acc], acc_ph);
      tc_fence_after();
      const int row = mb * 2 * BM + rank * BM + wq * 32 + lane;
      const uint32_t taddr = tmem_base + ((uint32_t)(wq * 32) << 16) + acc * BNT;
      if constexpr (RT) {
        if (ksp > 1) {
          epilogue_tile<EPI, BNT, F8>(args, taddr, row, nb, ksp, t, PartSrc{}, part * CW, (part + 1) * CW);
        } else {
          uint8_t* wst = rt_stg + wq * RT_WARP_BYTES;
          uint64_t* rb = rt_bar + wq * 2;
          const int r0w = mb * 2 * BM + rank * BM + wq * 32;
          const bool xo = args.xg_out != nullptr;
          auto load = [&](int c) {  // residual box of chunk c into buffer c & 1
            if (lane == 0) {
              bulk_wait_read<0>();  // the store that last read this buffer is done with it
              mbar_arrive_expect_tx(&rb[c & 1], 4096);
              tma_load_2d(wst + (c & 1) * 4096, &map_r, &rb[c & 1], nb * BNT + c * 32, r0w);
            }
          };
          load(0);
          load(1);
          float sq[2] = {0.f, 0.f};
#pragma unroll 1
          for (int c = 0; c < BNT / 32; ++c) {
            uint32_t r[32];
            tmem_ld32(taddr + c * 32, r);
            tmem_ld_wait();
            dequant32<F8>(args, (F8 && row < args.M) ? args.a_scale[row] : 0.f, nb * BNT + c * 32, r);
            mbar_wait(&rb[c & 1], (uint32_t)rt_ph[c & 1]);
            rt_ph[c & 1] ^= 1;
            float4* rowp = reinterpret_cast<float4*>(wst + (c & 1) * 4096 + lane * 128);
            uint32_t* xgp = reinterpret_cast<uint32_t*>(wst + 8192 + (c & 1) * 2048 + lane * 64);
            const float4* g4 = reinterpret_cast<const float4*>(args.g_next + nb * BNT + c * 32);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              float4 v = rowp[q ^ (lane & 7)];
              v.x += __uint_as_float(r[4 * q + 0]);
              v.y += __uint_as_float(r[4 * q + 1]);
              v.z += __uint_as_float(r[4 * q + 2]);
              v.w += __uint_as_float(r[4 * q + 3]);
              rowp[q ^ (lane & 7)] = v;
              if (xo) {
                const float4 g = g4[q];
                xgp[2 * q] = pack_bf16(v.x * g.x, v.y * g.y);
                xgp[2 * q + 1] = pack_bf16(v.z * g.z, v.w * g.w);
                sq[c >> 2] += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
              }
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&map_r, wst + (c & 1) * 4096, nb * BNT + c * 32, r0w);
              if (xo) tma_store_2d(&map_xo, wst + 8192 + (c & 1) * 2048, nb * BNT + c * 32, r0w);
              bulk_commit();
            }
            if (c + 2 < BNT / 32) load(c + 2);
          }
          if (xo && args.ss_out && row < args.M) {
            args.ss_out[(long long)row * args.ss_nseg + nb * 2] = sq[0];
            args.ss_out[(long long)row * args.ss_nseg + nb * 2 + 1] = sq[1];
          }
        }
      } else {
        epilogue_tile<EPI, BNT, F8>(args, taddr, row, nb, ksp, t, PartSrc{}, part * CW, (part + 1) * CW);
      }
      tc_fence_before();
      named_bar_sync(1, 128 * EW);
      if (threadIdx.x == 128) mbar_arrive_cluster(tempty0 + acc * 8);
    }
    if (RT && lane == 0) bulk_wait_all();  // residual / xg stores complete before the grid does
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 2 * BNT);
  }
}

// Work units of a reduce row: one per output quad, except that a RoPE unit covers a quad of a head's first 64 columns
// together with its rotation partner at +64, and a SiLU.mul unit a gate quad together with its up quad at +16, so no
// lane of a warp idles on the partner columns (the kernel is issue-bound at short M).
__host__ __device__ __forceinline__ int reduce_units_per_row(int epi, int N, int rope_cols) {
  return epi == EPI_QKV_ROPE ? rope_cols / 8 + (N - rope_cols) / 4 : epi == EPI_SILU_MUL ? N / 8 : N / 4;
}
template <int EPI>
__device__ __forceinline__ int reduce_unit_col(const GemmArgs& a, int u) {
  if constexpr (EPI == EPI_QKV_ROPE) {
    const int ru = a.rope_cols / 8;
    return u < ru ? (u >> 4) * 128 + (u & 15) * 4 : a.rope_cols + (u - ru) * 4;
  } else if constexpr (EPI == EPI_SILU_MUL) {
    return (u >> 2) * 32 + (u & 3) * 4;
  } else {
    return u * 4;
  }
}

// Grid-stride loop over output quads; IDX = int when M * N / 4 fits (32-bit row/column divisions: the 64-bit ones are
// a ~70-instruction software sequence each, three per quad, in a kernel that is issue-bound at short M)
template <int EPI, typename IDX>
__device__ __forceinline__ void splitk_reduce_loop(const GemmArgs& a, IDX total, IDX ncol4) {
  const size_t slice = (size_t)a.M * a.N;
  constexpr bool NORM = EPI == EPI_SILU_MUL || EPI == EPI_QKV_ROPE;
  // folded-norm consumers: the 1/rms of the block's rows (a block's quads span few rows) is computed once per row by
  // one warp - every segment sum loaded at once, then summed in segment order (row_inv_rms's order, so the result is
  // the same) - instead of by every thread through four dependent load batches
  __shared__ float s_ss[8][64];
  __shared__ float s_sc[8];
  const bool share = NORM && a.ss_in && a.ss_nseg <= 64;
  for (IDX base = (IDX)blockIdx.x * blockDim.x; base < total; base += (IDX)gridDim.x * blockDim.x) {
    const IDX i = base + threadIdx.x;
    const int r_first = static_cast<int>(base / ncol4);
    const IDX last = base + (IDX)blockDim.x - 1 < total ? base + (IDX)blockDim.x - 1 : total - 1;
    const int nrows = static_cast<int>(last / ncol4) - r_first + 1;
    const bool use = share && nrows <= 8;  // uniform across the block
    if (use) {
      const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
      if (w < nrows) {
        const float* src = a.ss_in + (long long)(r_first + w) * a.ss_nseg;
        for (int k = ln; k < a.ss_nseg; k += 32) s_ss[w][k] = __ldcg(src + k);
        __syncwarp();
        if (ln == 0) {
          float sum = 0.f;
#pragma unroll 16
          for (int k = 0; k < a.ss_nseg; ++k) sum += s_ss[w][k];  // loads batched ahead of the in-order adds
          s_sc[w] = rsqrtf(sum / a.norm_dim + a.norm_eps);
        }
      }
      __syncthreads();
    }
    if (i < total) {
      const int row = static_cast<int>(i / ncol4);
      const int col = reduce_unit_col<EPI>(a, static_cast<int>(i - (IDX)row * ncol4));
      int splits = a.k_splits;
      const float* p = a.split_ws + (size_t)row * a.N + col;
      if (a.sk_red) {  // stream-K partials: this column tile's contributors (gemm_sk.cu reduce mode)
        const int t = col / 256;
        splits = stream_owner(a.sk_w, a.sk_p, t * a.sk_nk + a.sk_nk - 1) - stream_owner(a.sk_w, a.sk_p, t * a.sk_nk) + 1;
      }
      splitk_reduce_quad<EPI>(a, row, col, p, slice, splits, use ? s_sc[row - r_first] : -1.f);
    }
    if (use) __syncthreads();  // s_ss / s_sc are rewritten by the next iteration
  }
}

template <int EPI>
__global__ void splitk_reduce_kernel(const GemmArgs a) {
  pdl_wait();
  pdl_trigger();
  const long long ncol4 = reduce_units_per_row(EPI, a.N, a.rope_cols);  // units per row
  const long long total = (long long)a.M * ncol4;
  if (total + 2LL * 148 * 8 * 256 < 0x7fffffffLL)  // base + stride stays below 2^31 too
    splitk_reduce_loop<EPI, int>(a, (int)total, (int)ncol4);
  else
    splitk_reduce_loop<EPI, long long>(a, total, ncol4);
}

int splitk_reduce_launch(int epi, const GemmArgs& args, cudaStream_t stream) {
  const long long total = (long long)args.M * reduce_units_per_row(epi, args.N, args.rope_cols);
  const int blocks = (int)((total + 255) / 256 < 148 * 8 ? (total + 255) / 256 : 148 * 8);
  switch (epi) {
    case EPI_BF16: launch_pdl(splitk_reduce_kernel<EPI_BF16>, dim3(blocks), dim3(256), 0, stream, args); break;
    case EPI_RESID_F32: launch_pdl(splitk_reduce_kernel<EPI_RESID_F32>, dim3(blocks), dim3(256), 0, stream, args); break;
    case EPI_SILU_MUL: launch_pdl(splitk_reduce_kernel<EPI_SILU_MUL>, dim3(blocks), dim3(256), 0, stream, args); break;
    case EPI_QKV_ROPE: launch_pdl(splitk_reduce_kernel<EPI_QKV_ROPE>, dim3(blocks), dim3(256), 0, stream, args); break;
    case EPI_F32: launch_pdl(splitk_reduce_kernel<EPI_F32>, dim3(blocks), dim3(256), 0, stream, args); break;
    default: return -3;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

int make_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t row_stride_bytes,
                      uint32_t box_inner, uint32_t box_outer) {
  auto fn = encode_fn();
  if (!fn) return -1;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

int make_tmap_3d_bf16(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t stride1_bytes,
                      uint64_t stride2_bytes, uint32_t b0, uint32_t b1, uint32_t b2) {
  auto fn = encode_fn();
  if (!fn) return -1;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

// 4-D map (d0 innermost, 128B swizzle), e.g. the prefix pool as [slot][layer][block_tokens][kv_dim] with boxes that
// take one layer of several consecutive slots.
int make_tmap_4d_bf16(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t d3,
                      uint64_t stride1_bytes, uint64_t stride2_bytes, uint64_t stride3_bytes, uint32_t b0, uint32_t b1,
                      uint32_t b2, uint32_t b3) {
  auto fn = encode_fn();
  if (!fn) return -1;
  cuuint64_t dims[4] = {d0, d1, d2, d3};
  cuuint64_t strides[3] = {stride1_bytes, stride2_bytes, stride3_bytes};
  cuuint32_t box[4] = {b0, b1, b2, b3};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

// Plain (unswizzled) 3-D map for epilogue stores: dims {d0, d1, d2}, strides in bytes, fp32 or bf16 elements.
int make_tmap_store_3d(CUtensorMap* map, const void* base, bool f32, uint64_t d0, uint64_t d1, uint64_t d2,
                       uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t b0, uint32_t b1) {
  auto fn = encode_fn();
  if (!fn) return -1;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
  cuuint32_t box[3] = {b0, b1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                  const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

// 2-D map for the RT epilogue: 32 x 32 boxes over an fp32 (128-byte swizzle) or bf16 (no swizzle) [rows, cols] matrix
int make_tmap_2d_epi(CUtensorMap* map, const void* base, bool f32, uint64_t cols, uint64_t rows, uint64_t row_stride_bytes,
                     bool swizzle128) {
  auto fn = encode_fn();
  if (!fn) return -1;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                  const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

int make_tmap_a(CUtensorMap* map, const void* A, long long lda, long long rows, int K) {
  return make_tmap_2d_bf16(map, A, K, rows, lda * 2, BK, BM);
}
int make_tmap_b(CUtensorMap* map, const void* B, long long ldb, int N, int K) {
  return make_tmap_2d_bf16(map, B, K, N, ldb * 2, BK, BN);
}
int make_tmap_b64(CUtensorMap* map, const void* B, long long ldb, int N, int K) {
  return make_tmap_2d_bf16(map, B, K, N, ldb * 2, BK, BN / 4);
}

int gemm_plan(GemmPlan* plan, const void* A, long long lda, const void* B, long long ldb, int M, int N, int K) {
  if (M <= 0 || N % BN != 0 || K % BK != 0) return -3;
  plan->M = M;
  plan->N = N;
  plan->K = K;
  plan->A = A;
  plan->lda = lda;
  if (make_tmap_2d_bf16(&plan->map_a, A, K, M, lda * 2, BK, BM)) return -2;
  if (make_tmap_2d_bf16(&plan->map_b, B, K, N, ldb * 2, BK, BN)) return -2;
  if (make_tmap_2d_bf16(&plan->map_b2, B, K, N, ldb * 2, BK, BM)) return -2;
  if (make_tmap_2d_bf16(&plan->map_b3, B, K, N, ldb * 2, BK, BM / 2)) return -2;
  return 0;
}

static void split_plan(int M, int N, int K, int* splits, int* kbps) {
  const int tiles_mn = ((M + BM - 1) / BM) * (N / BN);
  const int nk = K / BK;
  int s = 1;
  if (tiles_mn * 2 <= num_sms() && nk >= 16) {
    s = num_sms() / tiles_mn;
    s = s < nk / 8 ? s : nk / 8;
    s = s > 1 ? s : 1;
  }
  *kbps = (nk + s - 1) / s;
  *splits = (nk + *kbps - 1) / *kbps;
}

bool gemm_pair_narrow(int M, int N);

size_t gemm_split_ws_bytes(int M, int N, int K) {
  int s, kbps;
  split_plan(M, N, K, &s, &kbps);
  // pair kernel (M > 128): splits bounded by SM pairs / pair tiles (narrow 256 x 128 tiles for small M)
  const int tiles_mn = ((M + 2 * BM - 1) / (2 * BM)) * (N / (gemm_pair_narrow(M, N) ? 128 : BN));
  const int nk = K / BK;
  int s2 = 1;
  if (tiles_mn * 2 <= num_sms() / 2 && nk >= 16) {
    s2 = (num_sms() / 2) / tiles_mn;
    s2 = s2 < nk / 8 ? s2 : nk / 8;
    s2 = s2 > 1 ? s2 : 1;
  }
  const int smax = s > s2 ? s : s2;
  return smax > 1 ? (size_t)smax * M * N * sizeof(float) : 0;
}

template <int EPI, int BNT, bool F8 = false>
static int launch_pair_t(const CUtensorMap& map_a, const CUtensorMap& map_b2, const GemmArgs& in,
                         cudaStream_t stream) {
  ensure_smem_attr<gemm2_kernel<EPI, BNT, F8>>(pair_smem<EPI, BNT, F8>());
  GemmArgs args = in;
  args.k_splits = 1;
  const int tiles_mn = ((args.M + 2 * BM - 1) / (2 * BM)) * (args.N / BNT);
  if (args.split_ws) {
    // pair tiles: split K while fewer than SM-pairs/2 tiles exist (small-M prefix-hit GEMMs)
    const int nk = args.K / (F8 ? 2 * BK : BK);
    int s = 1;
    const int pairs = num_sms() / 2;
    if (tiles_mn * 2 <= pairs && nk >= 16) {
      s = pairs / tiles_mn;
      s = s < nk / 8 ? s : nk / 8;
      s = s > 1 ? s : 1;
    }
    if (s > 1) {
      args.k_splits = s;
      args.kb_per_split = (nk + s - 1) / s;
      args.k_splits = (nk + args.kb_per_split - 1) / args.kb_per_split;
      if ((size_t)args.k_splits * args.M * args.N * sizeof(float) > args.split_ws_bytes) args.k_splits = 1;
    }
  }
  const int tiles = tiles_mn * args.k_splits;
  const int npairs = tiles < num_sms() / 2 ? tiles : num_sms() / 2;
  // RT: residual / folded-norm-input maps over this launch's rows (32 x 32 boxes; rows >= M clipped by TMA)
  CUtensorMap map_r{}, map_xo{};
  if constexpr (pair_rt<EPI, BNT, F8>()) {
    if (args.k_splits == 1) {
      if (make_tmap_2d_epi(&map_r, args.resid, true, args.N, args.M, (uint64_t)args.ldr * 4, true) ||
          (args.xg_out && make_tmap_2d_epi(&map_xo, args.xg_out, false, args.N, args.M, (uint64_t)args.ldxg * 2, false)))
        return -2;
    }
  }
  launch_pdl(gemm2_kernel<EPI, BNT, F8>, dim3(2 * npairs), dim3(pair_threads<pair_ew<F8, BNT>()>()),
             pair_smem<EPI, BNT, F8>(), stream, map_a, map_b2, map_r, map_xo, args);
  if (args.k_splits > 1) {
    const long long total = (long long)args.M * reduce_units_per_row(EPI, args.N, args.rope_cols);
    const int blocks = (int)((total + 255) / 256 < 148 * 8 ? (total + 255) / 256 : 148 * 8);
    launch_pdl(splitk_reduce_kernel<EPI>, dim3(blocks), dim3(256), 0, stream, args);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

// 256 x 128 pair tiles when one row-tile of 256 x 256 tiles would leave most SM pairs idle (prefix hits)
bool gemm_pair_narrow(int M, int N) {
  // 256 x 128 pair tiles without split-K, or (default) 256 x 256 tiles + split-K: the wide tiles halve the activation
  // re-reads per weight byte and measured 2% faster per prefix hit. PO_PAIR_NARROW=1 selects the narrow tiles.
  static int mode = -1;
  if (mode < 0) {
    const char* v = getenv("PO_PAIR_NARROW");
    mode = (v && v[0] == '1') ? 1 : 0;
  }
  return mode && M <= 2 * BM && N / BN < num_sms() / 2 && N % 128 == 0;
}

// Raster group for a pair launch: m-blocks (256 rows) per sweep over N. The group's A rows should stay in L2 while B
// streams past them: 16 blocks of a K = 4096 operand are 32 MB, but the down projection's K = 14336 makes 16 blocks
// 117 MB (the whole L2), and ncu showed its A re-streamed (2.8x the algorithmic reads). Long-K launches therefore
// take PO_GROUP_LONGK blocks (default 8: 58 MB of A). The default for K <= 8192 stays 16.
static int pair_group(int K, int N) {
  static int longk = -1, widen = -1;
  if (longk < 0) {
    const char* v = getenv("PO_GROUP_LONGK");
    longk = v ? atoi(v) : 8;
    if (longk < 1) longk = 16;
    const char* w = getenv("PO_GROUP_WIDEN");  // A/B: m-blocks per sweep for wide launches (N >= 16384, gate/up)
    widen = w ? atoi(w) : 0;
  }
  if (K > 8192) return longk;
  if (widen > 0 && N >= 16384) return widen;
  return GROUP_M;
}

template <int EPI>
static int launch_pair(const CUtensorMap& map_a, const CUtensorMap& map_b2, const CUtensorMap* map_b3,
                       const GemmArgs& in0, cudaStream_t stream) {
  GemmArgs in = in0;
  if (in.group_m <= 0) in.group_m = pair_group(in.K, in.N);
  if (map_b3 && gemm_pair_narrow(in.M, in.N)) return launch_pair_t<EPI, 128>(map_a, *map_b3, in, stream);
  return launch_pair_t<EPI, 256>(map_a, map_b2, in, stream);
}

template <int EPI>
static int launch(const CUtensorMap& map_a, const CUtensorMap& map_b, const GemmArgs& in, cudaStream_t stream) {
  ensure_smem_attr<gemm_kernel<EPI>>(SMEM_BYTES);
  GemmArgs args = in;
  args.k_splits = 1;
  if (args.split_ws) {
    int s, kbps;
    split_plan(args.M, args.N, args.K, &s, &kbps);
    if (s > 1 && (size_t)s * args.M * args.N * sizeof(float) <= args.split_ws_bytes) {
      args.k_splits = s;
      args.kb_per_split = kbps;
    }
  }
  const int tiles = ((args.M + BM - 1) / BM) * (args.N / BN) * args.k_splits;
  const int grid = tiles < num_sms() ? tiles : num_sms();
  launch_pdl(gemm_kernel<EPI>, dim3(grid), dim3(NUM_THREADS), SMEM_BYTES, stream, map_a, map_b, args);
  if (args.k_splits > 1) {
    const long long total = (long long)args.M * reduce_units_per_row(EPI, args.N, args.rope_cols);
    const int blocks = (int)((total + 255) / 256 < 148 * 8 ? (total + 255) / 256 : 148 * 8);
    launch_pdl(splitk_reduce_kernel<EPI>, dim3(blocks), dim3(256), 0, stream, args);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

int gemm_launch_pair(const CUtensorMap& map_a, const CUtensorMap& map_b2, int epi, const GemmArgs& args,
                     cudaStream_t stream, const CUtensorMap* map_b3) {
  if (args.M <= 0) return 0;
  if (args.N % BN || args.K % BK) return -3;
  switch (epi) {
    case EPI_BF16: return launch_pair<EPI_BF16>(map_a, map_b2, map_b3, args, stream);
    case EPI_RESID_F32: return launch_pair<EPI_RESID_F32>(map_a, map_b2, map_b3, args, stream);
    case EPI_SILU_MUL: return launch_pair<EPI_SILU_MUL>(map_a, map_b2, map_b3, args, stream);
    case EPI_QKV_ROPE: return launch_pair<EPI_QKV_ROPE>(map_a, map_b2, map_b3, args, stream);
    case EPI_F32: return launch_pair<EPI_F32>(map_a, map_b2, map_b3, args, stream);
    default: return -3;
  }
}

// ------------------------------------------------------------------ FP8 (E4M3, W8A8)
int make_tmap_a_f8(CUtensorMap* map, const void* A, long long lda, long long rows, int K) {
  auto fn = encode_fn();
  if (!fn) return -1;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)lda};
  cuuint32_t box[2] = {2 * BK, BM};  // 128 bytes x 128 rows, the bf16 box geometry
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(A), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

size_t gemm_split_ws_bytes_f8(int M, int N, int K) {
  const int tiles_mn = ((M + 2 * BM - 1) / (2 * BM)) * (N / BN);
  const int nk = K / (2 * BK);
  int s = 1;
  if (tiles_mn * 2 <= num_sms() / 2 && nk >= 16) {
    s = (num_sms() / 2) / tiles_mn;
    s = s < nk / 8 ? s : nk / 8;
    s = s > 1 ? s : 1;
  }
  return s > 1 ? (size_t)s * M * N * sizeof(float) : 0;
}

int gemm_launch_pair_f8(const CUtensorMap& map_a, const CUtensorMap& map_b2, int epi, const GemmArgs& args,
                        cudaStream_t stream) {
  if (args.M <= 0) return 0;
  if (args.N % BN || args.K % (2 * BK) || !args.a_scale || !args.b_scale) return -3;
  switch (epi) {
    case EPI_BF16: return launch_pair_t<EPI_BF16, 256, true>(map_a, map_b2, args, stream);
    case EPI_RESID_F32: return launch_pair_t<EPI_RESID_F32, 256, true>(map_a, map_b2, args, stream);
    case EPI_SILU_MUL: return launch_pair_t<EPI_SILU_MUL, 256, true>(map_a, map_b2, args, stream);
    case EPI_QKV_ROPE: return launch_pair_t<EPI_QKV_ROPE, 256, true>(map_a, map_b2, args, stream);
    case EPI_F32: return launch_pair_t<EPI_F32, 256, true>(map_a, map_b2, args, stream);
    default: return -3;
  }
}

// One CTA per row: amax over the row (8 bf16 per 16-byte load), then e4m3 = satfinite_rn(x * 448 / amax).
__global__ void __launch_bounds__(256) quantize_rows_kernel(const __nv_bfloat16* __restrict__ x, long long ldx, int cols,
                                                            uint8_t* __restrict__ q, long long ldq,
                                                            float* __restrict__ scale) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[8];
  const int row = blockIdx.x;
  const uint4* src = reinterpret_cast<const uint4*>(x + (long long)row * ldx);
  const int nv = cols / 8;
  float amax = 0.f;
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    const uint4 v = src[i];
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[k]));
      amax = fmaxf(amax, fmaxf(fabsf(f.x), fabsf(f.y)));
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = amax;
  __syncthreads();
  amax = red[0];
#pragma unroll
  for (int k = 1; k < 8; ++k) amax = fmaxf(amax, red[k]);
  const float inv = amax > 0.f ? 448.f / amax : 0.f;
  if (threadIdx.x == 0) scale[row] = amax / 448.f;
  uint2* dst = reinterpret_cast<uint2*>(q + (long long)row * ldq);
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    const uint4 v = src[i];
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t o[2];
#pragma unroll
    for (int k = 0; k < 4; k += 2) {
      const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[k]));
      const float2 f1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[k + 1]));
      const uint32_t lo = __nv_cvt_float2_to_fp8x2(make_float2(f0.x * inv, f0.y * inv), __NV_SATFINITE, __NV_E4M3);
      const uint32_t hi = __nv_cvt_float2_to_fp8x2(make_float2(f1.x * inv, f1.y * inv), __NV_SATFINITE, __NV_E4M3);
      o[k / 2] = lo | (hi << 16);
    }
    dst[i] = make_uint2(o[0], o[1]);
  }
}

int quantize_rows_e4m3(const __nv_bfloat16* x, long long ldx, int rows, int cols, uint8_t* q, long long ldq,
                       float* scale, cudaStream_t stream) {
  if (rows <= 0) return 0;
  if (cols % 16 || ldx % 8 || ldq % 16) return -3;
  launch_pdl(quantize_rows_kernel, dim3(rows), dim3(256), 0, stream, x, ldx, cols, q, ldq, scale);
  return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

int gemm_launch(const CUtensorMap& map_a, const CUtensorMap& map_b, int epi, const GemmArgs& args,
                cudaStream_t stream) {
  if (args.M <= 0) return 0;
  if (args.N % BN || args.K % BK) return -3;
  switch (epi) {
    case EPI_BF16: return launch<EPI_BF16>(map_a, map_b, args, stream);
    case EPI_RESID_F32: return launch<EPI_RESID_F32>(map_a, map_b, args, stream);
    case EPI_SILU_MUL: return launch<EPI_SILU_MUL>(map_a, map_b, args, stream);
    case EPI_QKV_ROPE: return launch<EPI_QKV_ROPE>(map_a, map_b, args, stream);
    case EPI_F32: return launch<EPI_F32>(map_a, map_b, args, stream);
    default: return -3;
  }
}

bool gemm_use_pair(int M) {
  static int force_1cta = -1;
  if (force_1cta < 0) {
    const char* v = getenv("PO_GEMM_1CTA");
    force_1cta = (v && v[0] == '1') ? 1 : 0;
  }
  return !force_1cta && M > BM;
}

int gemm_run(const GemmPlan& plan, int epi, const GemmArgs& in, cudaStream_t stream) {
  GemmArgs args = in;
  args.M = plan.M;
  args.N = plan.N;
  args.K = plan.K;
  if (gemm_swap_enabled() && args.M <= 256) {
    if (args.sk_ws && gemm_sk_enabled(epi)) {
      const int rc = gemm_launch_sk(plan.map_b2, plan.A, plan.lda, epi, args, stream);
      if (rc != 1) return rc;
    }
    const int rc = gemm_launch_swap(plan.map_b2, plan.A, plan.lda, epi, args, stream);
    if (rc != 1) return rc;
  }
  if (gemm_use_pair(args.M)) return gemm_launch_pair(plan.map_a, plan.map_b2, epi, args, stream, &plan.map_b3);
  return gemm_launch(plan.map_a, plan.map_b, epi, args, stream);
}

}  // namespace po
