// Persistent weight-streaming layer kernel (see stream.cuh for the design).
//
// CTA pair layout (cluster of 2, 256 threads per CTA, one CTA per SM, grid = all SMs):
//   warp 0      TMA producer (one lane): per k-block its CTA's 128 activation rows + 128 of the 256 weight rows
//   warp 1      MMA issuer (leader CTA, one lane): tcgen05.mma.cta_group::2 M256 N256 K16 into a TMEM accumulator
//   warp 2      TMEM allocator (2 x 256 columns, double buffered across units and phases)
//   warps 4..7  epilogue: fused epilogue from TMEM, or fp32 partial dump + flag and the cooperative fix-up of the
//               split tiles; grid-barrier arrival after each phase
#include "stream.cuh"
#include "gemm_epi.cuh"

namespace po {

namespace {
constexpr int BM = 128;                        // rows per CTA (pair tile: 256)
constexpr int BN = 256;                        // weight rows (output columns) per pair tile
constexpr int BK = 64;
constexpr int HALF = 128 * BK * 2;             // 16 KB: 128 rows x 64 bf16 (A half or B half per CTA)
constexpr int STAGE = 2 * HALF;
constexpr int STAGES = 6;
constexpr int SMEM = STAGES * STAGE + 1024 + 256;
constexpr int NT = 256;

struct Geo {
  int nk, ntiles, spt, M, P;  // P: pairs with work (min(pairs, W): every one of them owns >= 1 k-block)
  long long W;
};
__device__ __forceinline__ Geo geo_of(const StreamPhase& p, int pairs) {
  Geo g;
  g.nk = p.g.K / BK;
  g.ntiles = p.g.N / BN;
  g.W = (long long)g.nk * g.ntiles;
  g.P = g.W < pairs ? (int)g.W : pairs;
  g.spt = p.slots_per_tile;
  g.M = p.g.M;
  return g;
}
__device__ __forceinline__ int range_lo(const Geo& g, int pair) {
  return pair < g.P ? stream_pair_start(g.W, g.P, pair) : (int)g.W;
}
__device__ __forceinline__ int range_hi(const Geo& g, int pair) {
  return pair < g.P ? stream_pair_start(g.W, g.P, pair + 1) : (int)g.W;
}
struct Unit {
  int tile, kb0, kb1, seg, nseg;
};
// The unit of pair `pair` that starts at global k-block kb (ends at its range end or the tile end).
__device__ __forceinline__ Unit unit_at(const Geo& g, int pair, int kb) {
  Unit u;
  u.tile = kb / g.nk;
  const int t0 = u.tile * g.nk;
  const int end = min(range_hi(g, pair), t0 + g.nk);
  u.kb0 = kb - t0;
  u.kb1 = end - t0;
  const int first = stream_owner(g.W, g.P, t0);
  u.seg = pair - first;
  u.nseg = stream_owner(g.W, g.P, t0 + g.nk - 1) - first + 1;
  return u;
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// generic-proxy writes of other CTAs (epilogue stores) -> this CTA's async-proxy reads (TMA), and the reverse
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

}  // namespace

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT, 1) stream_kernel(const __grid_constant__ StreamArgs A) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * HALF;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = warp_id();
  const int lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  const int P = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    for (int f = 0; f < A.nph; ++f) {
      tma_prefetch_desc(&A.ph[f].a);
      tma_prefetch_desc(&A.ph[f].b);
    }
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
  if (warp == 2) tmem_alloc_pair(tmem_slot, 2 * BN);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // the producer streams phase 0's first weight k-blocks before waiting for the previous kernel (weights are
  // constant); everyone else waits now
  if (warp != 0) pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t full0 = mapa_shared(smem_u32(full_bar), 0);
      int s = 0;
      uint32_t ph = 0;
      for (int f = 0; f < A.nph; ++f) {
        const StreamPhase& F = A.ph[f];
        const Geo g = geo_of(F, P);
        const int lo = range_lo(g, pair), hi = range_hi(g, pair);
        int pend_s[STAGES], pend_k[STAGES];
        int npend = 0;
        bool open = false;
        for (int kb = lo; kb < hi; ++kb) {
          const int tile = kb / g.nk, kk = kb - tile * g.nk;
          mbar_wait(&empty_bar[s], ph ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&full_bar[s], 2 * STAGE);
          const uint32_t fb = full0 + s * 8;
          tma_load_2d_pair(sB + s * HALF, &F.b, fb, kk * BK, tile * BN + rank * (BN / 2));
          if (open) {
            tma_load_2d_pair(sA + s * HALF, &F.a, fb, kk * BK, F.g.a_row0 + rank * BM);
          } else {
            pend_s[npend] = s;
            pend_k[npend] = kk;
            ++npend;
            if (npend == STAGES || kb + 1 == hi) {
              // the activations of this phase are the previous phase's output: wait for every CTA's epilogue
              if (f == 0) {
                pdl_wait();
              } else {
                const unsigned long long target = A.bar_base + (unsigned long long)f * gridDim.x;
                while (ld_acquire_u64(A.bar) < target) __nanosleep(64);
              }
              fence_proxy_async_global();
              open = true;
              for (int i = 0; i < npend; ++i)
                tma_load_2d_pair(sA + pend_s[i] * HALF, &F.a, full0 + pend_s[i] * 8, pend_k[i] * BK,
                                 F.g.a_row0 + rank * BM);
              npend = 0;
            }
          }
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
        if (f == 0 && !open) pdl_wait();
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(2 * BM, BN);
      int s = 0;
      uint32_t ph = 0;
      int it = 0;
      for (int f = 0; f < A.nph; ++f) {
        const Geo g = geo_of(A.ph[f], P);
        const int hi = range_hi(g, pair);
        for (int kb = range_lo(g, pair); kb < hi; ++it) {
          const Unit u = unit_at(g, pair, kb);
          const int acc = it & 1;
          const uint32_t acc_ph = (it >> 1) & 1;
          mbar_wait(&tempty_bar[acc], acc_ph ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc * BN;
          for (int k = u.kb0; k < u.kb1; ++k) {
            mbar_wait(&full_bar[s], ph);
            tc_fence_after();
            const uint64_t adesc = sdesc_kmajor_sw128(smem_u32(sA + s * HALF));
            const uint64_t bdesc = sdesc_kmajor_sw128(smem_u32(sB + s * HALF));
#pragma unroll
            for (int j = 0; j < BK / 16; ++j)
              mma_bf16_ss_pair(d_tmem, adesc + 2 * j, bdesc + 2 * j, idesc, (k != u.kb0 || j) ? 1u : 0u);
            mma_commit_pair(&empty_bar[s], 0x3);
            if (++s == STAGES) { s = 0; ph ^= 1; }
          }
          mma_commit_pair(&tfull_bar[acc], 0x3);
          kb += u.kb1 - u.kb0;
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int wq = warp & 3;
    const int et = threadIdx.x - 128;  // 0..127 within the epilogue warps
    const uint32_t tempty0 = mapa_shared(smem_u32(tempty_bar), 0);
    const int row = rank * BM + wq * 32 + lane;  // accumulator row of this thread (single 256-row m tile)
    int it = 0;
    for (int f = 0; f < A.nph; ++f) {
      const StreamPhase& F = A.ph[f];
      const Geo g = geo_of(F, P);
      const uint32_t tag = A.tag * 8u + (uint32_t)f;
      const long long slot_elems = (long long)g.M * BN;
      int split_tiles[2], nsplit = 0;
      const int hi = range_hi(g, pair);
      for (int kb = range_lo(g, pair); kb < hi; ++it) {
        const Unit u = unit_at(g, pair, kb);
        kb += u.kb1 - u.kb0;
        const int acc = it & 1;
        const uint32_t acc_ph = (it >> 1) & 1;
        mbar_wait(&tfull_bar[acc], acc_ph);
        tc_fence_after();
        const uint32_t taddr = tmem_base + ((uint32_t)(wq * 32) << 16) + acc * BN;
        if (u.nseg > 1) {
          // a tile cut across pairs: dump this segment's fp32 partial and raise its flag; the segments' owners
          // reduce the tile together once all are in (below)
          const long long slot = (long long)u.tile * g.spt + u.seg;
          float* dst = A.ws + slot * slot_elems + (long long)row * BN;
#pragma unroll 1
          for (int c = 0; c < BN; c += 32) {
            uint32_t r[32];
            tmem_ld32(taddr + c, r);
            tmem_ld_wait();
            if (row < g.M) {
              float4* d4 = reinterpret_cast<float4*>(dst + c);
#pragma unroll
              for (int q = 0; q < 8; ++q)
                d4[q] = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                    __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
            }
          }
          tc_fence_before();
          named_bar_sync(1, 128);
          if (et == 0) {
            mbar_arrive_cluster(tempty0 + acc * 8);
            __threadfence();
            st_release_u32(A.flags + slot * 2 + rank, tag);
          }
          split_tiles[nsplit++] = u.tile;
        } else {
          // a whole tile in one unit: fused epilogue straight from TMEM
          switch (F.epi) {
            case EPI_RESID_F32: epilogue_tile<EPI_RESID_F32, BN>(F.g, taddr, row, u.tile, 1, 0); break;
            case EPI_SILU_MUL: epilogue_tile<EPI_SILU_MUL, BN>(F.g, taddr, row, u.tile, 1, 0); break;
            case EPI_QKV_ROPE: epilogue_tile<EPI_QKV_ROPE, BN>(F.g, taddr, row, u.tile, 1, 0); break;
            default: epilogue_tile<EPI_BF16, BN>(F.g, taddr, row, u.tile, 1, 0); break;
          }
          tc_fence_before();
          named_bar_sync(1, 128);
          if (et == 0) mbar_arrive_cluster(tempty0 + acc * 8);
        }
      }
      // cooperative fix-up of the split tiles this pair holds a segment of (at most two: its first and last unit):
      // the tile's 2 x nseg CTAs each sum every segment for an interleaved share of its rows, in segment order
      for (int i = 0; i < nsplit; ++i) {
        const int t = split_tiles[i];
        const int q0 = stream_owner(g.W, g.P, t * g.nk);
        const int nseg = stream_owner(g.W, g.P, t * g.nk + g.nk - 1) - q0 + 1;
        const long long slot0 = (long long)t * g.spt;
        if (et == 0) {
          const int ranks = g.M > BM ? 2 : 1;  // a CTA with no rows below M dumps nothing but still flags
          for (int j = 0; j < nseg; ++j)
            for (int r = 0; r < ranks; ++r)
              while (ld_acquire_u32(A.flags + (slot0 + j) * 2 + r) != tag) __nanosleep(32);
        }
        named_bar_sync(2, 128);
        const int workers = 2 * nseg, worker = 2 * (pair - q0) + rank;
        const int sub = et >> 6, c = (et & 63) * 4;  // two rows per pass; each warp one 128-column segment
        const float* base = A.ws + slot0 * slot_elems + c;
        for (int rr = 2 * worker + sub; rr < g.M; rr += 2 * workers) {
          const float* p = base + (long long)rr * BN;
          switch (F.epi) {
            case EPI_RESID_F32: splitk_reduce_quad<EPI_RESID_F32>(F.g, rr, t * BN + c, p, slot_elems, nseg); break;
            case EPI_SILU_MUL: splitk_reduce_quad<EPI_SILU_MUL>(F.g, rr, t * BN + c, p, slot_elems, nseg); break;
            case EPI_QKV_ROPE: splitk_reduce_quad<EPI_QKV_ROPE>(F.g, rr, t * BN + c, p, slot_elems, nseg); break;
            default: splitk_reduce_quad<EPI_BF16>(F.g, rr, t * BN + c, p, slot_elems, nseg); break;
          }
        }
      }
      // this CTA's outputs of phase f are stored: arrive on the grid barrier
      named_bar_sync(1, 128);
      if (et == 0) {
        fence_proxy_async_global();
        __threadfence();
        atomicAdd(A.bar, 1ull);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 2 * BN);
  }
}

// ------------------------------------------------------------------ host side
int stream_pairs() { return num_sms() / 2; }

// partial slots per tile: every segment of a split tile dumps (0 when no tile is split)
static int slots_per_tile(int N, int K) {
  const int nk = K / BK, ntiles = N / BN;
  const long long W = (long long)nk * ntiles;
  const int P = W < stream_pairs() ? (int)W : stream_pairs();
  int most = 1;
  for (int t = 0; t < ntiles; ++t) {
    const int nseg = stream_owner(W, P, (t + 1) * nk - 1) - stream_owner(W, P, t * nk) + 1;
    most = nseg > most ? nseg : most;
  }
  return most > 1 ? most : 0;
}

size_t stream_ws_bytes(int M, int N, int K) { return (size_t)(N / BN) * slots_per_tile(N, K) * M * BN * sizeof(float); }
size_t stream_flag_count(int N, int K) { return (size_t)(N / BN) * slots_per_tile(N, K) * 2; }

int stream_launch(StreamArgs& a, cudaStream_t stream) {
  if (a.nph <= 0 || a.nph > STREAM_MAX_PHASES) return -3;
  for (int f = 0; f < a.nph; ++f) {
    StreamPhase& p = a.ph[f];
    const GemmArgs& g = p.g;
    if (g.M <= 0 || g.M > 2 * BM || g.N % BN || g.K % BK) return -3;
    p.slots_per_tile = slots_per_tile(g.N, g.K);
    if (stream_ws_bytes(g.M, g.N, g.K) > a.ws_bytes || stream_flag_count(g.N, g.K) > a.n_flags) return -3;
  }
  ensure_smem_attr<stream_kernel>(SMEM);
  launch_pdl(stream_kernel, dim3(2 * stream_pairs()), dim3(NT), SMEM, stream, a);
  return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

}  // namespace po
